// Host side of the C ABI (include/forestcoll.h): communicators, NVLink peer
// mapping through CUDA IPC, plan tables, chunk planning and launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fc_internal.h"

namespace {

constexpr uint32_t kCommMagic = 0x4d4d4346;  // 'FCMM'
constexpr uint32_t kBufMagic = 0x46554246;   // 'FBUF'
constexpr int kMaxC = 2048;                  // flag slots per tree / slot (chunks per launch)
constexpr int kTreeCap = 256;
constexpr int kCeLocalCtas = 48;             // copy-engine path: CTAs of the local shard copy
constexpr int kSlotCap = 512;
constexpr size_t kCtlBytes = 256;

struct CommBlob {
  uint32_t magic;
  int32_t rank, nranks, pad;
  uint64_t ws_bytes, flags_off, flags_words, scratch_off, scratch_bytes;
  cudaIpcMemHandle_t handle;
};
struct BufBlob {
  uint32_t magic;
  int32_t rank;
  uint64_t offset, bytes;
  cudaIpcMemHandle_t handle;
};
constexpr size_t kHandleBytes = 192;
static_assert(sizeof(CommBlob) <= kHandleBytes, "blob size");
static_assert(sizeof(BufBlob) <= kHandleBytes, "blob size");

struct Mapping {
  cudaIpcMemHandle_t handle;
  char* base;
};
// A registered allocation (the whole cudaMalloc segment holding the buffer,
// cuMemGetAddressRange), mapped into every peer.  Keyed by the driver's
// process-unique buffer id, so a segment freed and re-allocated at the same
// address is recognised as new.  Tensors are never pinned: the number of
// registrations is bounded by the allocator's segments.
struct Reg {
  uintptr_t lo, hi;        // the local segment
  uintptr_t anchor;        // local buffer registered (local rank 0's pointer)
  unsigned long long seq;  // registration number: equal on every rank (collective calls)
  unsigned long long buffer_id;
  char* peer[FC_MAXR];     // peer r's registered buffer, mapped into this process
  long long peer_lo[FC_MAXR], peer_hi[FC_MAXR];  // peer r's segment around peer[r] (offsets)
};
struct Plan {
  bool loaded = false;
  int nranks = 0, k = 0, ntrees = 0, max_slot_units = 0, max_slots = 0, max_mult = 0;
  int max_ag_slot_units = 0, max_ag_slots = 0;
  long long active_total = 0;
  int* d_tasks[FC_MAXR] = {};
  int nact[FC_MAXR] = {}, nwait[FC_MAXR] = {}, lag_max[FC_MAXR] = {};
  int* d_os = nullptr;  // RS/AR: one-shot forest program (FC_OS_TREE_WORDS per tree)
  int os_ntrees = 0;
  int flags = 0;        // TH_FLAGS (FC_PLAN_ONEHOP)
};

typedef CUresult (*PFN_getRange)(CUdeviceptr*, size_t*, CUdeviceptr);
typedef CUresult (*PFN_ptrAttr)(void*, CUpointer_attribute, CUdeviceptr);

}  // namespace

struct fc_comm {
  int rank = 0, nranks = 0, device = 0, virt = 0, nlocal = 0, connected = 0;
  int local[FC_MAXR] = {};      // rank ids executed by this process (grid order)
  bool is_local[FC_MAXR] = {};
  size_t ws_bytes = 0, flags_off = 0, flags_words = 0, scratch_off = 0, scratch_bytes = 0;
  char* ws[FC_MAXR] = {};
  bool own[FC_MAXR] = {};
  std::vector<Mapping> maps;
  std::vector<Reg> regs;
  unsigned long long reg_seq = 0;
  Plan plans[3];
  int ctas_per_rank = 64;
  long long chunk_max = 256 << 10, chunk_min = 16 << 10, items_per_worker = 4;
  long long timeout_ms = 120000;  // FORESTCOLL_TIMEOUT_MS overrides (default_ctas)
  int lag = 64;
  int copy_mode = 1;
  int dma_root_copy = 0;
  int worker_warps = 8;
  int pdl = 1;
  int proto = -1;                  // -1 auto, 0 chunk flags, 1 LL128
  long long ll_chunk_max = 64 << 10;
  int ll_worker_warps = 4;
  long long ll_max = 512LL << 20;  // auto: LL128 when bytes moved per rank <= this (and staging fits)
  int chunk_tail = 4;              // chunk-flag protocol: halving tail chunks per slice
  cudaStream_t side = nullptr;
  // NVLS pool (multicast object bound to a per-rank physical allocation)
  unsigned long long nvls_mc = 0, nvls_mem = 0;
  char* nvls_mc_va = nullptr;
  char* nvls_uc_va = nullptr;
  size_t nvls_bytes = 0;
  int nvls_bound = 0;
  int nvls_ctas = 32;
  long long nvls_ll_max = -1;         // NVLS allgather: LL multicast up to this output size
                                      // (-1: max(2 MiB, N x 512 KiB), measured crossover)
  long long nvls_ll_half = 0;         // LL staging half (2 halves reserved at the pool top)
  long long oneshot_ag_max = -1;      // tree engine: one-shot allgather up to this output size
                                      // (-1: 16 MiB; 0: off)
  long long oneshot_max = -1;         // tree engine: one-shot allreduce up to this many bytes
                                      // (-1: 2 MiB; reduce-scatter 2/N of it; 0: off)
  long long nvls_ll_red_max = -1;     // NVLS allreduce via LL multicast up to this many bytes
                                      // (-1: N x 64 KiB; reduce-scatter: 1/N of it)
  long long twohop_max = -1;          // tree engine: two-hop reductions up to this many input
                                      // bytes per rank (-1: default; 0: off)
  long long ce_min = -1;              // 2-rank forest: copy-engine allgather from this output
                                      // size (-1: 24 MiB; 0: off)
  int sm_count = 148;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_last = nullptr;     // cross-stream ordering of this comm's collectives
  cudaStream_t last_stream = nullptr;
  bool have_last = false;
  FcTraceRec* trace = nullptr;
  unsigned* trace_count = nullptr;
  unsigned trace_cap = 0;
  std::string err;
  long long info[8] = {};
};

namespace {

int fail(fc_comm* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define FC_CUDA(c, call)                                                                 \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail((c), FC_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));    \
  } while (0)

int esize_of(int dtype) {
  switch (dtype) {
    case FC_INT8: case FC_UINT8: return 1;
    case FC_FLOAT16: case FC_BFLOAT16: return 2;
    case FC_INT32: case FC_UINT32: case FC_FLOAT32: return 4;
    case FC_INT64: case FC_UINT64: case FC_FLOAT64: return 8;
    default: return 0;
  }
}

int reduce_kind(int dtype) {
  switch (dtype) {
    case FC_FLOAT32: return FC_FLOAT32;
    case FC_BFLOAT16: return FC_BFLOAT16;
    case FC_FLOAT16: return FC_FLOAT16;
    case FC_INT32: case FC_UINT32: return FC_INT32;
    default: return -1;
  }
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int alloc_workspace(fc_comm* c, char** out) {
  FC_CUDA(c, cudaMalloc((void**)out, c->ws_bytes));
  FC_CUDA(c, cudaMemset(*out, 0, c->scratch_off));  // control block + flags
  // LL128 staging lives in its own zeroed region: a line's flag word only ever
  // holds 0 or an epoch of this communicator, so a stale line can never match
  FC_CUDA(c, cudaMemset(*out + c->scratch_off + c->scratch_bytes, 0, c->scratch_bytes));
  return FC_SUCCESS;
}

int setup_layout(fc_comm* c, size_t scratch_bytes) {
  c->flags_off = kCtlBytes;
  c->flags_words = FC_READY_WORDS + kTreeCap + (size_t)(kTreeCap + kSlotCap) * kMaxC +
                   2 * FC_MAXR +     // + NVLS entry/exit barrier words
                   2 * FC_CE_SLOTS;  // + copy-engine path slots (64-bit)
  c->scratch_off = align_up(c->flags_off + c->flags_words * 4, 4096);
  c->scratch_bytes = align_up(scratch_bytes, 4096);
  c->ws_bytes = c->scratch_off + 2 * c->scratch_bytes;  // reduction scratch + LL128 staging
  return FC_SUCCESS;
}

PFN_getRange get_range_fn() {
  static PFN_getRange fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_getRange)p;
  }
  return fn;
}

PFN_ptrAttr ptr_attr_fn() {
  static PFN_ptrAttr fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_ptrAttr)p;
  }
  return fn;
}

// The allocation (segment) holding p: base, size and process-unique buffer id.
bool segment_of(const void* p, uintptr_t* base, size_t* size, unsigned long long* id) {
  PFN_getRange range = get_range_fn();
  PFN_ptrAttr attr = ptr_attr_fn();
  if (!range || !attr) return false;
  CUdeviceptr b = 0;
  size_t n = 0;
  if (range(&b, &n, (CUdeviceptr)p) != CUDA_SUCCESS) return false;
  unsigned long long bid = 0;
  if (attr(&bid, CU_POINTER_ATTRIBUTE_BUFFER_ID, (CUdeviceptr)p) != CUDA_SUCCESS) return false;
  *base = (uintptr_t)b;
  *size = n;
  *id = bid;
  return true;
}

int open_mapping(fc_comm* c, const cudaIpcMemHandle_t& h, char** base) {
  for (auto& m : c->maps)
    if (memcmp(&m.handle, &h, sizeof(h)) == 0) {
      *base = m.base;
      return FC_SUCCESS;
    }
  void* p = nullptr;
  FC_CUDA(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  c->maps.push_back(Mapping{h, (char*)p});
  *base = (char*)p;
  return FC_SUCCESS;
}

// The live registration covering [p, p + bytes), or null.  A registration
// whose segment was freed and its address range reused is stale (buffer id
// differs) and dropped.
const Reg* find_reg(fc_comm* c, const void* p, size_t bytes) {
  const uintptr_t a = (uintptr_t)p;
  for (size_t i = 0; i < c->regs.size(); ++i) {
    const Reg& r = c->regs[i];
    if (a < r.lo || a + bytes > r.hi) continue;
    if (c->virt) return &r;
    uintptr_t base;
    size_t size;
    unsigned long long id;
    if (segment_of(p, &base, &size, &id) && id == r.buffer_id) return &r;
    c->regs.erase(c->regs.begin() + i);  // stale
    return nullptr;
  }
  return nullptr;
}

// Collectives of one communicator share its control block, flags and scratch,
// so they execute one at a time.  Calls on one stream are ordered by that
// stream (and keep programmatic dependent launch between them: nothing is
// enqueued between two calls).  A call issued on another stream (FSDP's
// all-gather and reduce-scatter streams, say) first waits for an event
// recorded at that moment on the previous call's stream.  Issue order is the
// same on every rank of an SPMD program, so every rank runs the same sequence
// (the ordering NCCL keeps per communicator).  Inside CUDA-graph capture the
// graph's own edges order the calls.
bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
}

int order_begin(fc_comm* c, cudaStream_t s) {
  if (c->have_last && s != c->last_stream && !capturing(s) && !capturing(c->last_stream)) {
    if (cudaEventRecord(c->ev_last, c->last_stream) == cudaSuccess)
      FC_CUDA(c, cudaStreamWaitEvent(s, c->ev_last, 0));
    else
      (void)cudaGetLastError();  // that stream is gone: its work has been retired
  }
  return FC_SUCCESS;
}

int order_end(fc_comm* c, cudaStream_t s) {
  if (capturing(s)) return FC_SUCCESS;
  c->last_stream = s;
  c->have_last = true;
  return FC_SUCCESS;
}

// Tree-engine one-shot launches (fc_nvls.cu, modes 6/7/8): one grid serves
// every local rank; several local ranks (virtual mode) launch cooperatively
// with all CTAs co-resident.
int oneshot_common(fc_comm* c, FcNvlsParams& P, int mode, int rd, const void* const* sends,
                   void* const* recvs, long long half, void* stream) {
  P.nranks = c->nranks;
  P.rank = c->local[0];
  P.mode = mode;
  P.dtype = rd;
  P.scale = 1.0f / (float)c->nranks;
  for (int r = 0; r < c->nranks; ++r) P.peer_stage[r] = c->ws[r] + c->scratch_off + c->scratch_bytes;
  P.ll_half = half;
  P.timeout_ns = c->timeout_ms * 1000000LL;
  P.nlocal = c->nlocal;
  for (int i = 0; i < c->nlocal; ++i) {
    P.lrank[i] = c->local[i];
    P.lctl[i] = (FcCtl*)c->ws[c->local[i]];
    P.lsend[i] = (const char*)sends[i];
    P.lout[i] = (char*)recvs[i];
  }
  if (c->nlocal == 1) {
    P.ctas_per_rank = c->sm_count;  // one CTA per SM: polls and tree evaluation
  } else {
    int maxc = 0;
    FC_CUDA(c, (cudaError_t)fc_oneshot_max_ctas(mode, rd, c->nranks, &maxc));
    P.ctas_per_rank = std::min(c->sm_count, maxc / c->nlocal);
    if (P.ctas_per_rank < 1)
      return fail(c, FC_ERR_UNSUPPORTED, "device cannot co-schedule %d one-shot ranks", c->nlocal);
  }
  {
    const int st = order_begin(c, (cudaStream_t)stream);
    if (st) return st;
  }
  const int e = fc_nvls_launch(P, P.nlocal * P.ctas_per_rank, stream);
  if (e) return fail(c, FC_ERR_CUDA, "one-shot launch failed: %s", cudaGetErrorString((cudaError_t)e));
  {
    const int st = order_end(c, (cudaStream_t)stream);
    if (st) return st;
  }
  c->info[0] = 1;
  c->info[1] = 1;
  c->info[3] = P.nlocal * P.ctas_per_rank;
  c->info[5] = 4;  // one-shot
  return FC_SUCCESS;
}

// One-shot reduce-scatter / allreduce for small inputs: every rank stores its
// whole input as LL128 lines into every rank's staging through the peer
// mappings, then evaluates the forest's in-trees locally in the executor's
// order (bit-identical to the forest kernel).  One hop instead of RS depth +
// AG depth.
int run_oneshot(fc_comm* c, int coll, const Plan& pl, const void* const* sends,
                void* const* recvs, long long S, long long total, int es, int rd, int op,
                long long half, void* stream, bool twohop = false) {
  FcNvlsParams P;
  memset(&P, 0, sizeof(P));
  P.op = op;
  P.os_trees = pl.d_os;
  P.os_ntrees = pl.os_ntrees;
  P.k = pl.k;
  P.buf_bytes = total * es;
  P.count = total;
  P.shard_elems = S;
  const int mode = twohop ? (coll == FC_REDUCE_SCATTER ? 10 : 9) : (coll == FC_REDUCE_SCATTER ? 6 : 7);
  const int st = oneshot_common(c, P, mode, rd, sends, recvs, half, stream);
  if (!st && twohop) c->info[5] = 7;  // two-hop
  return st;
}

// One-hop allgather (fc_oneshot_ag128_kernel): outputs are written locally
// only, so no buffer registration is used.
int run_oneshot_ag(fc_comm* c, const void* const* sends, void* const* recvs,
                   long long shard_bytes, long long half, void* stream) {
  FcNvlsParams P;
  memset(&P, 0, sizeof(P));
  P.shard_bytes = shard_bytes;
  return oneshot_common(c, P, 8, FC_FLOAT32, sends, recvs, half, stream);
}

// Copy-engine allgather of the 2-rank single-switch forest (fc_ce.cu): the
// tree of root r is the edge r -> peer, executed as one cudaMemcpyAsync of
// the own shard into the peer's registered output between two handshake
// kernels; the own shard is placed by an SM copy kernel on the side stream.
int run_ce_ag(fc_comm* c, const void* send, void* recv, long long shard_bytes, void* stream) {
  const int me = c->rank, peer = 1 - c->rank;
  const long long total = 2 * shard_bytes;
  const Reg* reg = find_reg(c, recv, (size_t)total);
  if (!reg)
    return fail(c, FC_ERR_NOT_REGISTERED,
                "output buffer %p (%lld bytes) is not registered (fc_buffer_register)", recv, total);
  const long long delta = (long long)((uintptr_t)recv - reg->anchor);
  if (delta < reg->peer_lo[peer] || delta + total > reg->peer_hi[peer])
    return fail(c, FC_ERR_INVALID_ARG, "output at offset %lld exceeds the peer's registered segment",
                delta);
  char* peer_out = reg->peer[peer] + delta;
  FcCeParams P;
  memset(&P, 0, sizeof(P));
  P.ctl = (FcCtl*)c->ws[me];
  const size_t ce_off = c->flags_off + (c->flags_words - 2 * FC_CE_SLOTS) * 4;
  P.my_slots = (unsigned long long*)(c->ws[me] + ce_off);
  P.peer_slots = (unsigned long long*)(c->ws[peer] + ce_off);
  P.tag = (reg->seq * 0x9E3779B97F4A7C15ull) ^ ((unsigned long long)delta * 0xC2B2AE3D27D4EB4Full) ^
          (unsigned long long)total;
  P.timeout_ns = c->timeout_ms * 1000000LL;
  P.me = me;
  P.peer = peer;
  const cudaStream_t s = (cudaStream_t)stream;
  {
    const int st = order_begin(c, s);
    if (st) return st;
  }
  char* own_out = (char*)recv + (size_t)me * shard_bytes;
  const bool local = own_out != (const char*)send;
  // own shard -> own output slot: an SM copy kernel on the side stream, run
  // concurrently with the copy engine.  kCeLocalCtas CTAs copy 2+ TB/s, well
  // ahead of the NVLink transfer; a full-GPU grid contends with the copy
  // engine for HBM and slows the whole call by 20 % (measured, N=2 1 GiB).
  if (local) {
    FC_CUDA(c, cudaEventRecord(c->ev_fork, s));
    FC_CUDA(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    FC_CUDA(c, (cudaError_t)fc_ce_copy_launch(own_out, send, shard_bytes, kCeLocalCtas, c->side));
    FC_CUDA(c, cudaEventRecord(c->ev_join, c->side));
  }
  P.phase = 0;
  FC_CUDA(c, (cudaError_t)fc_ce_sync_launch(P, stream));
  FC_CUDA(c, cudaMemcpyAsync(peer_out + (size_t)me * shard_bytes, send, (size_t)shard_bytes,
                             cudaMemcpyDeviceToDevice, s));
  P.phase = 1;
  FC_CUDA(c, (cudaError_t)fc_ce_sync_launch(P, stream));
  if (local) FC_CUDA(c, cudaStreamWaitEvent(s, c->ev_join, 0));
  {
    const int st = order_end(c, s);
    if (st) return st;
  }
  c->info[0] = local ? 3 : 2;  // kernels launched
  c->info[1] = 1;
  c->info[2] = 1;
  c->info[3] = 1;
  c->info[5] = 5;  // copy engine
  return FC_SUCCESS;
}

// Run one collective over this comm's local ranks.  With `path_out` set,
// only decide: store the path the call would take (0 chunk flags, 1 LL128,
// 4 one-hop / one-shot) and launch nothing (fc_call_path).
int run(fc_comm* c, int coll, const void* const* sends, void* const* recvs, size_t count,
        int dtype, int op, void* stream, int* path_out = nullptr, long long scratch_cap = 0,
        long long* scratch_need = nullptr) {
  if (!c) return FC_ERR_INVALID_ARG;
  if (!c->virt && !c->connected)
    return fail(c, FC_ERR_INVALID_ARG, "communicator is not connected (fc_comm_connect)");
  Plan& pl = c->plans[coll];
  if (!pl.loaded) return fail(c, FC_ERR_PLAN, "no plan loaded for collective %d", coll);
  const int es = esize_of(dtype);
  if (!es) return fail(c, FC_ERR_INVALID_ARG, "unknown dtype %d", dtype);
  int rd = FC_FLOAT32;
  if (coll != FC_ALLGATHER) {
    rd = reduce_kind(dtype);
    if (rd < 0) return fail(c, FC_ERR_UNSUPPORTED, "dtype %d cannot be reduced", dtype);
    if (op != FC_SUM && op != FC_AVG)
      return fail(c, FC_ERR_UNSUPPORTED, "reduction op %d unsupported", op);
    if (op == FC_AVG && rd == FC_INT32)
      return fail(c, FC_ERR_UNSUPPORTED, "AVG is implemented for floating-point dtypes only");
  }
  const int N = c->nranks;
  long long S, stride, total;
  if (coll == FC_ALLREDUCE) {
    const long long a = FC_ALIGN / es;
    S = ((long long)count + N - 1) / N;
    S = (S + a - 1) / a * a;
    stride = S;
    total = (long long)count;
  } else {
    S = (long long)count;
    stride = S;
    total = S * N;
  }
  if (path_out) *path_out = -1;  // nothing to move
  else c->info[0] = c->info[1] = c->info[2] = c->info[3] = 0;
  if (total == 0) return FC_SUCCESS;
  for (int i = 0; i < c->nlocal && !path_out; ++i)
    if (!sends[i] || !recvs[i]) return fail(c, FC_ERR_INVALID_ARG, "null buffer");

  // The 1-rank forest (N=1 is outside the reference's API, topology.py:263-266)
  // is its root's copy send -> recv: one full-GPU vector copy kernel
  if (N == 1 && coll == FC_ALLGATHER && c->nlocal == 1) {
    if (path_out) return *path_out = 6, FC_SUCCESS;
    {
      const int st = order_begin(c, (cudaStream_t)stream);
      if (st) return st;
    }
    const bool copy = recvs[0] != sends[0];
    if (copy)
      FC_CUDA(c, (cudaError_t)fc_ce_copy_launch(recvs[0], sends[0], total * es, 2 * c->sm_count,
                                                stream));
    {
      const int st = order_end(c, (cudaStream_t)stream);
      if (st) return st;
    }
    c->info[0] = copy ? 1 : 0;
    c->info[1] = c->info[2] = 1;
    c->info[3] = 2 * c->sm_count;
    c->info[5] = 6;  // local copy
    return FC_SUCCESS;
  }
  // Every choice below depends only on values that are equal on every rank
  // (sizes, dtype, plan, options): ranks must run the same kernel.  Local
  // buffer alignment is handled inside the kernels (ld_u64_any/st_u64_any).
  // scratch_need (fc_call_scratch): decide as if the workspace held
  // scratch_cap bytes per region and report what the chosen path needs
  const long long scratch = scratch_need ? scratch_cap : (long long)c->scratch_bytes;
  const long long half = scratch / 2 / 4096 * 4096;
  auto decided = [&](int path, long long need) {
    *path_out = path;
    if (scratch_need) *scratch_need = need;
    return FC_SUCCESS;
  };
  if (scratch_need) *scratch_need = 0;
  const bool onehop = (pl.flags & FC_PLAN_ONEHOP) != 0 && c->proto < 0;
  // 2-rank single-switch forest: each tree is one edge, moved by the copy
  // engine (fc_ce.cu) from ce_min output bytes (the peer's output must be
  // registered, as for the chunk-flag protocol)
  if (coll == FC_ALLGATHER && onehop && N == 2 && !c->virt && c->nlocal == 1 && c->ce_min != 0) {
    // measured vs the LL128 forest at N=2 (tools/exp_n2_ag_mid.sh): +3 % at
    // 24 MiB, +11 % at 32 MiB, +4 % at 96 MiB, +9 % at 1 GiB, +12 % at 4 GiB
    // (0.856 of T*); below 24 MiB the one-hop path or the forest wins
    const long long lim = c->ce_min > 0 ? c->ce_min : (24LL << 20);
    if (total * es >= lim) {
      if (path_out) return decided(5, 0);
      return run_ce_ag(c, sends[0], recvs[0], S * es, stream);
    }
  }
  // small allgathers on a single-switch forest: one hop (every root stores
  // its shard into every peer's LL128 staging) instead of the forest's depth;
  // same per-link load (FC_PLAN_ONEHOP).  A forced protocol is honoured.
  if (coll == FC_ALLGATHER && onehop && c->oneshot_ag_max != 0) {
    const long long bytes = total * es;  // output bytes
    // measured crossover vs the forest's LL128 at N=4: between 16 and 32 MiB
    const long long lim = c->oneshot_ag_max > 0 ? c->oneshot_ag_max : (16LL << 20);
    const long long lines = (S * es + 119) / 120;
    // any shard length: a partial last word travels zero-padded in its line
    if (bytes <= lim && (long long)N * lines * 128 <= half) {
      if (path_out) return decided(4, 2 * (long long)N * lines * 128);
      return run_oneshot_ag(c, sends, recvs, S * es, half, stream);
    }
  }
  // small reductions: one-shot (one hop) instead of the forest's two chains
  if (coll != FC_ALLGATHER && onehop && pl.d_os && c->oneshot_max != 0) {
    const long long bytes = total * es;  // per-rank input bytes (AR: buffer; RS: N shards)
    // measured crossover vs the forest kernel at N=4: allreduce 2 MiB,
    // reduce-scatter 2 x that / N of input
    const long long lim = c->oneshot_max > 0 ? c->oneshot_max : (2LL << 20);
    const long long lines = (bytes + 119) / 120;
    if (bytes <= (coll == FC_REDUCE_SCATTER ? 2 * lim / N : lim) && bytes % 8 == 0 &&
        (S * es) % 8 == 0 && (long long)N * lines * 128 <= half) {
      if (path_out) return decided(4, 2 * (long long)N * lines * 128);
      return run_oneshot(c, coll, pl, sends, recvs, S, total, es, rd, op, half, stream);
    }
  }
  // mid-size reductions: two hops (shards to their roots, reduced shards to
  // everyone; fc_nvls.cu fc_twohop128_kernel) -- the forest's link loads,
  // two hops instead of the in-trees' plus out-trees' depths
  if (coll != FC_ALLGATHER && onehop && pl.d_os && c->twohop_max != 0) {
    const long long bytes = total * es;
    // measured crossover vs the LL128 forest (tools/exp_twohop_r02.sh): N=4
    // allreduce 4 MiB +56 %, 8 MiB +17 %, 16 MiB even; N=2 4 MiB +15 %, 8 MiB
    // -6 %.  Reduce-scatter (input bytes) crosses over at 2/3 of that.
    const long long lim = c->twohop_max > 0 ? c->twohop_max : (N <= 2 ? (6LL << 20) : (12LL << 20));
    const long long need = 2LL * N * ((S * es + 119) / 120) * 128;  // hop-1 + hop-2 lines
    if (bytes <= (coll == FC_REDUCE_SCATTER ? 2 * lim / 3 : lim) && bytes % 8 == 0 &&
        (S * es) % 8 == 0 && need <= half) {
      if (path_out) return decided(7, 2 * need);
      return run_oneshot(c, coll, pl, sends, recvs, S, total, es, rd, op, half, stream, true);
    }
  }
  FcParams P;
  memset(&P, 0, sizeof(P));
  P.nranks = N;
  P.nlocal = c->nlocal;
  P.k = pl.k;
  for (int r = 0; r < N; ++r) {
    P.scratch[r] = c->ws[r] + c->scratch_off;
    P.flags[r] = (unsigned*)(c->ws[r] + c->flags_off);
  }
  for (int i = 0; i < c->nlocal; ++i) {
    const int r = c->local[i];
    P.local_rank[i] = r;
    P.tasks[i] = pl.d_tasks[i];
    P.nactive[i] = pl.nact[i];
    P.nwait[i] = pl.nwait[i];
    P.lag_max[i] = pl.lag_max[i];
    P.ctl[i] = (FcCtl*)c->ws[r];
    P.send[r] = (const char*)sends[i];
    P.recv[r] = (char*)recvs[i];
  }
  P.shard_elems = S;
  P.stride_elems = stride;
  P.total_elems = total;
  P.esize = es;
  P.dtype = dtype;
  P.op = op;
  P.scale = 1.0f / (float)c->nranks;
  P.maxc = kMaxC;
  P.cnt_off = FC_READY_WORDS;
  P.ag_flag_off = FC_READY_WORDS + kTreeCap;
  P.rs_flag_off = P.ag_flag_off + kTreeCap * kMaxC;
  P.timeout_ns = c->timeout_ms * 1000000LL;
  P.ctas_per_rank = c->ctas_per_rank;
  P.lag = c->lag;
  P.copy_mode = c->copy_mode;
  P.worker_warps = c->worker_warps;
  P.pdl = c->pdl;
  P.trace = c->trace;
  P.trace_count = c->trace_count;
  P.trace_cap = c->trace_cap;

  // Protocol and chunk plan: identical on every rank (they depend only on S,
  // dtype, the plan and the options, which must match across ranks).
  const long long slice_unit = (S + pl.k - 1) / pl.k * es;  // bytes per unit of multiplicity
  const long long max_slice = slice_unit * pl.max_mult;
  const long long avg_active = std::max(1LL, pl.active_total / N);
  auto chunks_for = [&](long long chunk_max, int ww) {
    const long long workers = (long long)c->ctas_per_rank * (fc_warps_per_cta() / ww);
    long long n = (max_slice + chunk_max - 1) / chunk_max;
    n = std::max(n, (c->items_per_worker * workers + avg_active - 1) / avg_active);
    n = std::min(n, std::max(1LL, max_slice / std::max(1LL, c->chunk_min)));
    return std::min(std::max(n, 1LL), 1LL << 30);
  };
  // LL128 (small/medium messages): single window, 8-byte aligned slices, and
  // staging for every in-edge of the call fits in scratch.
  int proto = 0;
  long long n = 0, W = 0;
  if (c->proto != 0) {
    // any slice length and offset works: a slice that is not a multiple of 8
    // bytes ends in a partial payload word (run_item_ll), and 4-byte aligned
    // slices keep batched 4-byte accesses.  Measured at N=4 against the chunk
    // flags: allreduce bf16 25 MiB + 1 element 317 vs 216 GB/s, reduce-scatter
    // fp32 256 MiB + 1 738 vs 376, allgather fp32 64 MiB + 1 622 vs 536.
    // Allgathers whose slices are not even 4-byte aligned (odd 2-byte counts)
    // would run the byte-granular loops and keep the chunk flags.
    bool aligned = (stride * es) % 4 == 0;  // slice offsets: rank-uniform
    for (int r = 0; r < N && aligned; ++r) {
      long long Sr = std::max(0LL, std::min(S, total - (long long)r * stride));
      for (int m = 0; m <= pl.k && aligned; ++m) aligned = ((Sr * m / pl.k) * es) % 4 == 0;
    }
    aligned = aligned || coll != FC_ALLGATHER || c->proto == 1;
    const long long unit_lines = (slice_unit + 119) / 120;
    const long long llu = unit_lines * 128;
    const long long rs_need = (long long)pl.max_slot_units * llu + 256LL * pl.max_slots;
    const long long ag_base = (rs_need + 255) / 256 * 256;
    const long long need = ag_base + (long long)pl.max_ag_slot_units * llu + 256LL * pl.max_ag_slots;
    const long long moved = (coll == FC_REDUCE_SCATTER) ? total * es : S * es * N;
    const bool want = c->proto == 1 || moved <= c->ll_max;
    // the LL region (scratch_bytes) is two halves used by alternate epochs
    if (aligned && want && need <= half) {
      proto = 1;
      if (scratch_need) *scratch_need = 2 * need;
      n = std::min<long long>(chunks_for(c->ll_chunk_max, c->ll_worker_warps), kMaxC);
      W = n;
      P.ll_unit_bytes = llu;
      P.ll_region_off = scratch;
      P.ll_half = half;
      P.ll_ag_base = ag_base;
      P.worker_warps = c->ll_worker_warps;
    } else if (c->proto == 1) {
      return fail(c, FC_ERR_UNSUPPORTED, "LL protocol forced but not applicable (alignment/scratch)");
    }
  }
  if (proto == 0) {
    n = chunks_for(c->chunk_max, c->worker_warps);
    W = std::min<long long>(n, kMaxC);
    // shrinking tail chunks (see chunk_bound in fc_device.cuh): only when the
    // slice has enough chunks that the halved ones stay >= chunk_min-ish
    int tail = 0;
    while (tail < c->chunk_tail && (n >> (tail + 1)) >= 8) ++tail;
    P.tail = tail;
    const long long wreg = 1LL << tail;
    const long long fsum = wreg * (n - tail) + wreg - 1;  // chunk_prefix(n, n, tail)
    auto unit_for = [&](long long w) {  // bytes of the widest window of w chunks, per unit
      return (long long)align_up((size_t)((slice_unit * w * wreg + fsum - 1) / fsum), FC_ALIGN);
    };
    if (coll != FC_ALLGATHER) {
      auto need = [&](long long w) {
        return (long long)pl.max_slot_units * unit_for(w) + 2LL * FC_ALIGN * pl.max_slots;
      };
      while (W > 1 && need(W) > scratch) W = std::max(1LL, W / 2);
      if (scratch_need) *scratch_need = need(W);
      if (need(W) > scratch && !scratch_need)
        return fail(c, FC_ERR_INVALID_ARG,
                    "scratch too small: %lld bytes needed per window, %zu available",
                    need(W), c->scratch_bytes);
      P.unit_bytes = unit_for(W);
    }
  }
  if (path_out) return decided(proto, scratch_need ? *scratch_need : 0);
  P.nchunks = (int)n;
  P.proto = proto;
  // the chunk-flag protocol stores into peers' outputs (AG recv, AR buf):
  // those must be registered; LL128 only writes peers' staging
  if (proto == 0 && !c->virt && coll != FC_REDUCE_SCATTER) {
    const size_t need = (size_t)total * es;
    const Reg* reg = find_reg(c, recvs[0], need);
    if (!reg)
      return fail(c, FC_ERR_NOT_REGISTERED,
                  "output buffer %p (%zu bytes) is not registered (fc_buffer_register)",
                  recvs[0], need);
    // peers' outputs sit at the same offset from their registered buffers
    // (SPMD allocation order); the tag below makes any rank that disagrees
    // fail loudly on the device before a single store lands
    const long long delta = (long long)((uintptr_t)recvs[0] - reg->anchor);
    for (int r = 0; r < N; ++r)
      if (!c->is_local[r]) P.recv[r] = reg->peer[r] + delta;
    // identity of the output every peer must be writing to in this call
    P.tag = (reg->seq * 0x9E3779B97F4A7C15ull) ^ ((unsigned long long)delta * 0xC2B2AE3D27D4EB4Full) ^
            (unsigned long long)need;
  }
  const int coop = c->nlocal > 1 ? 1 : 0;  // local ranks wait on each other in one grid
  int launches = 0, grid = 0;
  {
    const int st = order_begin(c, (cudaStream_t)stream);
    if (st) return st;
  }
  // allgather: a copy engine places each local root's own shard into its
  // output concurrently with the kernel (no SM bandwidth spent on it)
  bool dma = false;
  if (coll == FC_ALLGATHER && c->dma_root_copy) {
    FC_CUDA(c, cudaEventRecord(c->ev_fork, (cudaStream_t)stream));
    FC_CUDA(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    for (int i = 0; i < c->nlocal; ++i) {
      const int r = P.local_rank[i];
      char* dstp = P.recv[r] + (size_t)r * S * es;
      if (dstp != P.send[r])
        FC_CUDA(c, cudaMemcpyAsync(dstp, P.send[r], (size_t)S * es, cudaMemcpyDeviceToDevice,
                                   c->side));
    }
    FC_CUDA(c, cudaEventRecord(c->ev_join, c->side));
    P.root_local_done = 1;
    dma = true;
  }
  for (long long c0 = 0; c0 < n; c0 += W) {
    P.c0 = (int)c0;
    P.c1 = (int)std::min(n, c0 + W);
    // The claim-order skew only has to exceed the chunk span of the window to
    // keep every item's dependencies earlier in key order; a larger lag just
    // adds empty claims (stages x lag of them), which dominate tiny messages.
    P.lag = (int)std::min<long long>(c->lag, P.c1 - P.c0);
    const int e = fc_launch(P, rd, coop, stream, &grid);
    if (e != 0)
      return fail(c, FC_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString((cudaError_t)e));
    ++launches;
  }
  if (dma) FC_CUDA(c, cudaStreamWaitEvent((cudaStream_t)stream, c->ev_join, 0));
  {
    const int st = order_end(c, (cudaStream_t)stream);
    if (st) return st;
  }
  c->info[0] = launches;
  c->info[1] = n;
  c->info[2] = W;
  c->info[3] = grid;
  c->info[4] = P.unit_bytes;
  c->info[5] = proto;
  return FC_SUCCESS;
}

int free_plan(fc_comm* c, Plan& p) {
  for (int i = 0; i < FC_MAXR; ++i)
    if (p.d_tasks[i]) {
      cudaFree(p.d_tasks[i]);
      p.d_tasks[i] = nullptr;
    }
  if (p.d_os) {
    cudaFree(p.d_os);
    p.d_os = nullptr;
  }
  p.loaded = false;
  (void)c;
  return FC_SUCCESS;
}

int make_side_stream(fc_comm* c) {
  FC_CUDA(c, cudaEventCreateWithFlags(&c->ev_last, cudaEventDisableTiming));
  FC_CUDA(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  FC_CUDA(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  FC_CUDA(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  return FC_SUCCESS;
}

int default_ctas(fc_comm* c) {
  // a straggling rank (checkpoint I/O, data-loader stall) must not kill the
  // communicator: the device flag-wait timeout defaults to minutes
  if (const char* t = getenv("FORESTCOLL_TIMEOUT_MS")) {
    const long long v = atoll(t);
    if (v > 0) c->timeout_ms = v;
  }
  int per_sm = 0, sms = 0;
  FC_CUDA(c, (cudaError_t)fc_max_ctas_per_sm(FC_FLOAT32, &per_sm));
  int v = 0;
  for (int rd : {FC_BFLOAT16, FC_FLOAT16, FC_INT32}) {
    FC_CUDA(c, (cudaError_t)fc_max_ctas_per_sm(rd, &v));
    per_sm = std::min(per_sm, v);
  }
  FC_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  c->sm_count = sms;
  const int cap = per_sm * sms / c->nlocal;
  if (cap < 1) return fail(c, FC_ERR_UNSUPPORTED, "device cannot co-schedule %d ranks", c->nlocal);
  // virtual mode: every SM (one co-resident grid; 18 CTAs per rank at N=8 measured +2 %
  // over 16 on the N=1 bench workload, tools/exp_n1_r02.sh)
  c->ctas_per_rank = std::min(c->virt ? std::max(1, sms / c->nlocal) : 128, cap);
  c->worker_warps = c->virt ? 1 : 8;
  c->ll_worker_warps = c->virt ? 1 : 4;
  // virtual ranks share one HBM: LL staging doubles the traffic, so keep it for small calls
  if (c->virt) c->ll_max = 16LL << 20;
  // all ranks share one HBM and one grid: no drain to shorten (measured -1 % with tail 4)
  if (c->virt) c->chunk_tail = 0;
  // and finer chunks keep the depth-7 chains' fill and drain short (128 KiB: +1.5 %)
  if (c->virt) c->chunk_max = 128 << 10;
  return make_side_stream(c);
}

// -- driver entry points (no -lcuda: resolved through the runtime) ---------
struct Drv {
  CUresult (*getDevice)(CUdevice*, int);
  CUresult (*getAttr)(int*, CUdevice_attribute, CUdevice);
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t,
                        size_t, unsigned long long);
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
  CUresult (*exportHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                           unsigned long long);
  CUresult (*importHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                        unsigned long long);
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*memUnmap)(CUdeviceptr, size_t);
  CUresult (*memRelease)(CUmemGenericAllocationHandle);
  CUresult (*addrFree)(CUdeviceptr, size_t);
  bool ok = false;
};

const Drv& drv() {
  static Drv d;
  static bool tried = false;
  if (tried) return d;
  tried = true;
  auto get = [](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess;
  };
  d.ok = get("cuDeviceGet", (void**)&d.getDevice) &&
         get("cuDeviceGetAttribute", (void**)&d.getAttr) &&
         get("cuMulticastCreate", (void**)&d.mcCreate) &&
         get("cuMulticastAddDevice", (void**)&d.mcAddDevice) &&
         get("cuMulticastBindMem", (void**)&d.mcBindMem) &&
         get("cuMulticastUnbind", (void**)&d.mcUnbind) &&
         get("cuMulticastGetGranularity", (void**)&d.mcGranularity) &&
         get("cuMemExportToShareableHandle", (void**)&d.exportHandle) &&
         get("cuMemImportFromShareableHandle", (void**)&d.importHandle) &&
         get("cuMemCreate", (void**)&d.memCreate) &&
         get("cuMemAddressReserve", (void**)&d.addrReserve) && get("cuMemMap", (void**)&d.memMap) &&
         get("cuMemSetAccess", (void**)&d.setAccess) && get("cuMemUnmap", (void**)&d.memUnmap) &&
         get("cuMemRelease", (void**)&d.memRelease) && get("cuMemAddressFree", (void**)&d.addrFree);
  return d;
}

#define FC_DRV(c, call)                                                              \
  do {                                                                               \
    CUresult r_ = (call);                                                            \
    if (r_ != CUDA_SUCCESS) return fail((c), FC_ERR_CUDA, "%s failed (CUresult %d)", #call, (int)r_); \
  } while (0)

struct NvlsBlob {
  uint32_t magic;
  int32_t fd;  // POSIX file descriptor of the multicast object (valid in the holder)
  uint64_t bytes;
};
constexpr uint32_t kNvlsMagic = 0x534c564e;  // 'NVLS'
static_assert(sizeof(NvlsBlob) <= kHandleBytes, "nvls blob size");

CUmulticastObjectProp mc_prop(fc_comm* c, size_t bytes) {
  CUmulticastObjectProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.numDevices = (unsigned)c->nranks;
  prop.size = bytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return prop;
}

int run_nvls(fc_comm* c, int mode, const void* send, void* buf, void* out, size_t count, int dtype,
             int op, void* stream) {
  if (!c || !c->nvls_bound) return fail(c, FC_ERR_INVALID_ARG, "NVLS pool is not set up");
  const int es = esize_of(dtype);
  if (!es) return fail(c, FC_ERR_INVALID_ARG, "unknown dtype %d", dtype);
  int rd = FC_FLOAT32;
  if (mode != 0) {
    rd = reduce_kind(dtype);
    if (rd < 0) return fail(c, FC_ERR_UNSUPPORTED, "dtype %d cannot be reduced", dtype);
    if (op != FC_SUM && op != FC_AVG)
      return fail(c, FC_ERR_UNSUPPORTED, "reduction op %d unsupported", op);
    if (op == FC_AVG && rd == FC_INT32)
      return fail(c, FC_ERR_UNSUPPORTED, "AVG is implemented for floating-point dtypes only");
  }
  const uintptr_t b = (uintptr_t)buf, lo = (uintptr_t)c->nvls_uc_va;
  const int N = c->nranks;
  long long shard, total;
  if (mode == 2) {
    const long long a = FC_ALIGN / es;
    long long S = ((long long)count + N - 1) / N;
    S = (S + a - 1) / a * a;
    shard = S * es;
    total = (long long)count * es;
  } else {
    shard = (long long)count * es;
    total = shard * N;
  }
  if (total == 0) return FC_SUCCESS;
  const size_t usable = c->nvls_bytes - 2 * (size_t)c->nvls_ll_half;  // LL staging on top
  const long long ll_max =
      c->nvls_ll_max >= 0 ? c->nvls_ll_max : std::max<long long>(2LL << 20, N * (512LL << 10));
  // Engine choice from rank-uniform values only (sizes, options, plan): every
  // rank must run the same kernel.  The LL kernels move 8-byte units, so a
  // rank whose buffers are not 8-byte aligned fails loudly below instead of
  // silently taking another engine (the Python layer stages such views).
  if (mode == 0 && total <= ll_max && shard % 8 == 0 && 2LL * shard * N <= c->nvls_ll_half)
    mode = 3;  // LL over multicast: any device buffers
  // small reductions: LL multicast of the whole input + local tree evaluation
  // (needs the forest program of the loaded plan)
  // Every rank moves its whole input (N x a reduce-scatter's need), and the
  // local tree evaluation is compute: it pays off only for small buffers
  // (measured at N=4: allreduce up to 256 KiB, 1.6x the tree engine).
  const long long red_max =
      c->nvls_ll_red_max >= 0 ? c->nvls_ll_red_max : (long long)N * (64LL << 10);
  const Plan& rp = c->plans[mode == 1 ? FC_REDUCE_SCATTER : FC_ALLREDUCE];
  const long long red_lim = mode == 1 ? red_max / N : red_max;
  if ((mode == 1 || mode == 2) && rp.loaded && rp.d_os && total <= red_lim && total % 8 == 0 &&
      shard % 8 == 0 && 2LL * total * N <= c->nvls_ll_half)
    mode = mode == 1 ? 4 : 5;
  if (mode >= 3 && ((uintptr_t)buf % 8 || (send && (uintptr_t)send % 8) ||
                    (out && (uintptr_t)out % 8)))
    return fail(c, FC_ERR_INVALID_ARG,
                "NVLS LL path: buffers must be 8-byte aligned (the path is chosen from sizes "
                "alone, equal on every rank)");
  if (mode < 3) {
    if (b < lo || b + (size_t)total > lo + usable)
      return fail(c, FC_ERR_NOT_REGISTERED, "buffer %p is not inside the NVLS pool", buf);
    if ((b - lo) % 16 || shard % 16 || total % 16)
      return fail(c, FC_ERR_UNSUPPORTED, "NVLS needs 16-byte aligned shards");
  }
  FcNvlsParams P;
  memset(&P, 0, sizeof(P));
  P.nranks = N;
  P.rank = c->rank;
  P.mode = mode;
  P.dtype = rd;
  P.op = mode == 0 ? FC_SUM : op;
  P.scale = 1.0f / (float)N;
  P.bar_off = (int)(c->flags_words - 2 * FC_MAXR);
  P.ctl = (FcCtl*)c->ws[c->rank];
  for (int r = 0; r < N; ++r) P.flags[r] = (unsigned*)(c->ws[r] + c->flags_off);
  P.mc = c->nvls_mc_va + (b - lo);
  P.send = (const char*)send;
  P.out = (char*)out;
  if (mode >= 3) {
    P.mc_stage = c->nvls_mc_va + usable;
    P.uc_stage = c->nvls_uc_va + usable;
    P.ll_half = c->nvls_ll_half;
  }
  if (mode == 3) P.out = (char*)buf;
  if (mode >= 4) {  // reduce-scatter: send = buf (N shards) -> out; allreduce: buf in place
    P.send = (const char*)buf;
    P.out = mode == 4 ? (char*)out : (char*)buf;
    P.os_trees = rp.d_os;
    P.os_ntrees = rp.os_ntrees;
    P.k = rp.k;
    P.buf_bytes = total;
    P.count = total / es;
    P.shard_elems = shard / es;
  }
  P.shard_bytes = shard;
  P.total_bytes = total;
  P.timeout_ns = c->timeout_ms * 1000000LL;
  {
    const int st = order_begin(c, (cudaStream_t)stream);
    if (st) return st;
  }
  // LL modes poll and (for reductions) evaluate trees: one CTA per SM
  const int e = fc_nvls_launch(P, mode >= 3 ? c->sm_count : c->nvls_ctas, stream);
  if (e) return fail(c, FC_ERR_CUDA, "NVLS launch failed: %s", cudaGetErrorString((cudaError_t)e));
  {
    const int st = order_end(c, (cudaStream_t)stream);
    if (st) return st;
  }
  c->info[0] = 1;
  c->info[5] = mode >= 3 ? 3 : 2;  // engine: nvls (3: LL multicast)
  return FC_SUCCESS;
}

}  // namespace

extern "C" {

const char* fc_version(void) { return "forestcoll-b200 0.1.0 (sm_100a)"; }

size_t fc_handle_bytes(void) { return kHandleBytes; }

int fc_comm_init(int rank, int nranks, int device, size_t scratch_bytes, fc_comm_t** out) {
  if (!out || nranks < 1 || nranks > FC_MAXR || rank < 0 || rank >= nranks)
    return FC_ERR_INVALID_ARG;
  *out = nullptr;
  fc_comm* c = new fc_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  c->nlocal = 1;
  c->local[0] = rank;
  c->is_local[rank] = true;
  setup_layout(c, scratch_bytes);
  int st;
  if (cudaSetDevice(device) != cudaSuccess || (st = alloc_workspace(c, &c->ws[rank])) != 0 ||
      (st = default_ctas(c)) != 0) {
    if (c->ws[rank]) cudaFree(c->ws[rank]);
    fprintf(stderr, "fc_comm_init: %s\n", c->err.c_str());
    delete c;
    return FC_ERR_CUDA;
  }
  c->own[rank] = true;
  c->connected = (nranks == 1);
  *out = c;
  return FC_SUCCESS;
}

int fc_comm_init_ranks(const int* ranks, int nlocal, int nranks, int device,
                       size_t scratch_bytes, fc_comm_t** out) {
  if (!out || !ranks || nlocal < 1 || nranks < 1 || nranks > FC_MAXR || nlocal > nranks)
    return FC_ERR_INVALID_ARG;
  *out = nullptr;
  fc_comm* c = new fc_comm();
  c->nranks = nranks;
  c->device = device;
  c->nlocal = nlocal;
  c->rank = ranks[0];
  for (int i = 0; i < nlocal; ++i) {
    if (ranks[i] < 0 || ranks[i] >= nranks || c->is_local[ranks[i]]) {
      delete c;
      return FC_ERR_INVALID_ARG;
    }
    c->local[i] = ranks[i];
    c->is_local[ranks[i]] = true;
  }
  c->virt = nlocal == nranks ? 1 : 0;
  c->connected = c->virt;
  setup_layout(c, scratch_bytes);
  int st = cudaSetDevice(device) == cudaSuccess ? 0 : FC_ERR_CUDA;
  for (int i = 0; i < nlocal && st == 0; ++i) {
    st = alloc_workspace(c, &c->ws[c->local[i]]);
    if (st == 0) c->own[c->local[i]] = true;
  }
  if (st == 0) st = default_ctas(c);
  if (st != 0) {
    fprintf(stderr, "fc_comm_init_ranks: %s\n", c->err.c_str());
    for (int r = 0; r < FC_MAXR; ++r)
      if (c->own[r]) cudaFree(c->ws[r]);
    delete c;
    return st;
  }
  *out = c;
  return FC_SUCCESS;
}

int fc_comm_init_virtual(int nranks, int device, size_t scratch_bytes, fc_comm_t** out) {
  if (!out || nranks < 1 || nranks > FC_MAXR) return FC_ERR_INVALID_ARG;
  *out = nullptr;
  fc_comm* c = new fc_comm();
  c->nranks = nranks;
  c->device = device;
  c->virt = 1;
  c->nlocal = nranks;
  for (int r = 0; r < nranks; ++r) {
    c->local[r] = r;
    c->is_local[r] = true;
  }
  c->connected = 1;
  setup_layout(c, scratch_bytes);
  int st = cudaSetDevice(device) == cudaSuccess ? 0 : FC_ERR_CUDA;
  for (int r = 0; r < nranks && st == 0; ++r) {
    st = alloc_workspace(c, &c->ws[r]);
    if (st == 0) c->own[r] = true;
  }
  if (st == 0) st = default_ctas(c);
  if (st != 0) {
    fprintf(stderr, "fc_comm_init_virtual: %s\n", c->err.c_str());
    for (int r = 0; r < nranks; ++r)
      if (c->own[r]) cudaFree(c->ws[r]);
    delete c;
    return st;
  }
  *out = c;
  return FC_SUCCESS;
}

int fc_comm_export(fc_comm_t* c, void* handle) {
  if (!c || !handle || c->virt) return FC_ERR_INVALID_ARG;
  FC_CUDA(c, cudaSetDevice(c->device));
  for (int i = 0; i < c->nlocal; ++i) {  // one blob per local rank
    CommBlob b;
    memset(&b, 0, sizeof(b));
    b.magic = kCommMagic;
    b.rank = c->local[i];
    b.nranks = c->nranks;
    b.ws_bytes = c->ws_bytes;
    b.flags_off = c->flags_off;
    b.flags_words = c->flags_words;
    b.scratch_off = c->scratch_off;
    b.scratch_bytes = c->scratch_bytes;
    FC_CUDA(c, cudaIpcGetMemHandle(&b.handle, c->ws[c->local[i]]));
    char* dst = (char*)handle + (size_t)i * kHandleBytes;
    memset(dst, 0, kHandleBytes);
    memcpy(dst, &b, sizeof(b));
  }
  return FC_SUCCESS;
}

int fc_comm_connect(fc_comm_t* c, const void* handles) {
  if (!c || !handles || c->virt) return FC_ERR_INVALID_ARG;
  FC_CUDA(c, cudaSetDevice(c->device));
  for (int r = 0; r < c->nranks; ++r) {
    CommBlob b;
    memcpy(&b, (const char*)handles + (size_t)r * kHandleBytes, sizeof(b));
    if (b.magic != kCommMagic || b.rank != r || b.nranks != c->nranks)
      return fail(c, FC_ERR_INVALID_ARG, "bad communicator handle for rank %d", r);
    if (b.ws_bytes != c->ws_bytes || b.flags_off != c->flags_off ||
        b.scratch_off != c->scratch_off || b.scratch_bytes != c->scratch_bytes)
      return fail(c, FC_ERR_INVALID_ARG,
                  "rank %d workspace layout differs (scratch_bytes must match on all ranks)", r);
    if (c->is_local[r]) continue;
    char* base = nullptr;
    int st = open_mapping(c, b.handle, &base);
    if (st) return st;
    c->ws[r] = base;
  }
  c->connected = 1;
  return FC_SUCCESS;
}

int fc_comm_set_option(fc_comm_t* c, int option, long long v) {
  if (!c) return FC_ERR_INVALID_ARG;
  switch (option) {
    case FC_OPT_CTAS_PER_RANK: {
      int per_sm = 0, sms = 0;
      FC_CUDA(c, (cudaError_t)fc_max_ctas_per_sm(FC_FLOAT32, &per_sm));
      FC_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
      if (v < 1 || v * c->nlocal > (long long)per_sm * sms)
        return fail(c, FC_ERR_INVALID_ARG, "ctas_per_rank %lld out of range", v);
      c->ctas_per_rank = (int)v;
      return FC_SUCCESS;
    }
    case FC_OPT_CHUNK_MAX:
      if (v < 256) return fail(c, FC_ERR_INVALID_ARG, "chunk_max too small");
      c->chunk_max = v;
      return FC_SUCCESS;
    case FC_OPT_CHUNK_MIN:
      if (v < 16) return fail(c, FC_ERR_INVALID_ARG, "chunk_min too small");
      c->chunk_min = v;
      return FC_SUCCESS;
    case FC_OPT_ITEMS_PER_WORKER:
      if (v < 0) return fail(c, FC_ERR_INVALID_ARG, "items_per_worker < 0");
      c->items_per_worker = v;
      return FC_SUCCESS;
    case FC_OPT_TIMEOUT_MS:
      if (v < 1) return fail(c, FC_ERR_INVALID_ARG, "timeout must be positive");
      c->timeout_ms = v;
      return FC_SUCCESS;
    case FC_OPT_LAG:
      if (v < 0 || v > 4096) return fail(c, FC_ERR_INVALID_ARG, "lag out of range");
      c->lag = (int)v;
      return FC_SUCCESS;
    case FC_OPT_COPY_MODE:
      if (v < 0 || v > 1) return fail(c, FC_ERR_INVALID_ARG, "copy_mode is 0 or 1");
      c->copy_mode = (int)v;
      return FC_SUCCESS;
    case FC_OPT_DMA_ROOT_COPY:
      c->dma_root_copy = v ? 1 : 0;
      return FC_SUCCESS;
    case FC_OPT_WORKER_WARPS:
      if (v != 1 && v != 2 && v != 4 && v != 8)
        return fail(c, FC_ERR_INVALID_ARG, "worker_warps must be 1, 2, 4 or 8");
      c->worker_warps = (int)v;
      return FC_SUCCESS;
    case FC_OPT_PROTO:
      if (v < -1 || v > 1) return fail(c, FC_ERR_INVALID_ARG, "proto is -1 (auto), 0 or 1");
      c->proto = (int)v;
      return FC_SUCCESS;
    case FC_OPT_LL_MAX:
      if (v < 0) return fail(c, FC_ERR_INVALID_ARG, "ll_max < 0");
      c->ll_max = v;
      return FC_SUCCESS;
    case FC_OPT_PDL:
      c->pdl = v ? 1 : 0;
      return FC_SUCCESS;
    case FC_OPT_CHUNK_TAIL:
      if (v < 0 || v > 8) return fail(c, FC_ERR_INVALID_ARG, "chunk_tail out of range [0, 8]");
      c->chunk_tail = (int)v;
      return FC_SUCCESS;
    case FC_OPT_NVLS_LL_MAX:
      if (v < 0) return fail(c, FC_ERR_INVALID_ARG, "nvls_ll_max < 0");
      c->nvls_ll_max = v;
      return FC_SUCCESS;
    case FC_OPT_NVLS_LL_HALF:
      return fail(c, FC_ERR_INVALID_ARG, "nvls_ll_half is read-only");
    case FC_OPT_MAX_CTAS_PER_RANK:
      return fail(c, FC_ERR_INVALID_ARG, "max_ctas_per_rank is read-only");
    case FC_OPT_NVLS_LL_RED_MAX:
      if (v < 0) return fail(c, FC_ERR_INVALID_ARG, "nvls_ll_red_max < 0");
      c->nvls_ll_red_max = v;
      return FC_SUCCESS;
    case FC_OPT_ONESHOT_MAX:
      if (v < 0) return fail(c, FC_ERR_INVALID_ARG, "oneshot_max < 0");
      c->oneshot_max = v;
      return FC_SUCCESS;
    case FC_OPT_ONESHOT_AG_MAX:
      if (v < 0) return fail(c, FC_ERR_INVALID_ARG, "oneshot_ag_max < 0");
      c->oneshot_ag_max = v;
      return FC_SUCCESS;
    case FC_OPT_CE_MIN:
      if (v < 0) return fail(c, FC_ERR_INVALID_ARG, "ce_min < 0");
      c->ce_min = v;
      return FC_SUCCESS;
    case FC_OPT_TWOHOP_MAX:
      if (v < 0) return fail(c, FC_ERR_INVALID_ARG, "twohop_max < 0");
      c->twohop_max = v;
      return FC_SUCCESS;
    case FC_OPT_NVLS_CTAS:
      if (v < 1 || v > 1024) return fail(c, FC_ERR_INVALID_ARG, "nvls_ctas out of range");
      c->nvls_ctas = (int)v;
      return FC_SUCCESS;
    case FC_OPT_LL_CHUNK_MAX:
      if (v < 1024) return fail(c, FC_ERR_INVALID_ARG, "ll_chunk_max too small");
      c->ll_chunk_max = v;
      return FC_SUCCESS;
    case FC_OPT_LL_WORKER_WARPS:
      if (v != 1 && v != 2 && v != 4 && v != 8)
        return fail(c, FC_ERR_INVALID_ARG, "ll_worker_warps must be 1, 2, 4 or 8");
      c->ll_worker_warps = (int)v;
      return FC_SUCCESS;
    default:
      return fail(c, FC_ERR_INVALID_ARG, "unknown option %d", option);
  }
}

int fc_comm_get_option(fc_comm_t* c, int option, long long* v) {
  if (!c || !v) return FC_ERR_INVALID_ARG;
  switch (option) {
    case FC_OPT_CTAS_PER_RANK: *v = c->ctas_per_rank; return FC_SUCCESS;
    case FC_OPT_CHUNK_MAX: *v = c->chunk_max; return FC_SUCCESS;
    case FC_OPT_CHUNK_MIN: *v = c->chunk_min; return FC_SUCCESS;
    case FC_OPT_ITEMS_PER_WORKER: *v = c->items_per_worker; return FC_SUCCESS;
    case FC_OPT_TIMEOUT_MS: *v = c->timeout_ms; return FC_SUCCESS;
    case FC_OPT_LAG: *v = c->lag; return FC_SUCCESS;
    case FC_OPT_COPY_MODE: *v = c->copy_mode; return FC_SUCCESS;
    case FC_OPT_DMA_ROOT_COPY: *v = c->dma_root_copy; return FC_SUCCESS;
    case FC_OPT_WORKER_WARPS: *v = c->worker_warps; return FC_SUCCESS;
    case FC_OPT_PROTO: *v = c->proto; return FC_SUCCESS;
    case FC_OPT_LL_MAX: *v = c->ll_max; return FC_SUCCESS;
    case FC_OPT_LL_CHUNK_MAX: *v = c->ll_chunk_max; return FC_SUCCESS;
    case FC_OPT_NVLS_CTAS: *v = c->nvls_ctas; return FC_SUCCESS;
    case FC_OPT_PDL: *v = c->pdl; return FC_SUCCESS;
    case FC_OPT_CHUNK_TAIL: *v = c->chunk_tail; return FC_SUCCESS;
    case FC_OPT_NVLS_LL_MAX:
      *v = c->nvls_ll_max >= 0 ? c->nvls_ll_max
                               : std::max<long long>(2LL << 20, c->nranks * (512LL << 10));
      return FC_SUCCESS;
    case FC_OPT_NVLS_LL_HALF: *v = c->nvls_ll_half; return FC_SUCCESS;
    case FC_OPT_NVLS_LL_RED_MAX:
      *v = c->nvls_ll_red_max >= 0 ? c->nvls_ll_red_max : (long long)c->nranks * (64LL << 10);
      return FC_SUCCESS;
    case FC_OPT_ONESHOT_MAX:
      *v = c->oneshot_max >= 0 ? c->oneshot_max : (2LL << 20);
      return FC_SUCCESS;
    case FC_OPT_ONESHOT_AG_MAX:
      *v = c->oneshot_ag_max >= 0 ? c->oneshot_ag_max : (16LL << 20);
      return FC_SUCCESS;
    case FC_OPT_CE_MIN:
      *v = c->ce_min >= 0 ? c->ce_min : (24LL << 20);
      return FC_SUCCESS;
    case FC_OPT_TWOHOP_MAX:
      *v = c->twohop_max >= 0 ? c->twohop_max : (c->nranks <= 2 ? (6LL << 20) : (12LL << 20));
      return FC_SUCCESS;
    case FC_OPT_LL_WORKER_WARPS: *v = c->ll_worker_warps; return FC_SUCCESS;
    case FC_OPT_MAX_CTAS_PER_RANK: {
      int per_sm = 0;
      FC_CUDA(c, (cudaError_t)fc_max_ctas_per_sm(FC_FLOAT32, &per_sm));
      *v = (long long)per_sm * c->sm_count / c->nlocal;
      return FC_SUCCESS;
    }
    default: return fail(c, FC_ERR_INVALID_ARG, "unknown option %d", option);
  }
}

int fc_comm_check(fc_comm_t* c, int* device_error) {
  if (!c) return FC_ERR_INVALID_ARG;
  FC_CUDA(c, cudaSetDevice(c->device));
  FC_CUDA(c, cudaDeviceSynchronize());
  int worst = 0;
  for (int i = 0; i < c->nlocal; ++i) {
    const int r = c->local[i];
    FcCtl ctl;
    FC_CUDA(c, cudaMemcpy(&ctl, c->ws[r], sizeof(ctl), cudaMemcpyDeviceToHost));
    if (ctl.error && !worst) {
      worst = (int)ctl.error;
      if (ctl.error == FC_DEVERR_BUFFER_MISMATCH)
        fail(c, FC_ERR_DEVICE,
             "rank %d: device error %u (rank %u passed a different output buffer: every rank "
             "must pass the same registered buffer, offset and size)", r, ctl.error, ctl.info[0]);
      else
        fail(c, FC_ERR_DEVICE, "rank %d: device error %u (flag wait timed out; epoch %u, value %u)",
             r, ctl.error, ctl.info[1], ctl.info[2]);
    }
  }
  if (device_error) *device_error = worst;
  return worst ? FC_ERR_DEVICE : FC_SUCCESS;
}

int fc_comm_destroy(fc_comm_t* c) {
  if (!c) return FC_SUCCESS;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& p : c->plans) free_plan(c, p);
  for (auto& m : c->maps) cudaIpcCloseMemHandle(m.base);
  if (c->nvls_bound) {
    const Drv& d = drv();
    d.memUnmap((CUdeviceptr)c->nvls_mc_va, c->nvls_bytes);
    d.addrFree((CUdeviceptr)c->nvls_mc_va, c->nvls_bytes);
    d.memUnmap((CUdeviceptr)c->nvls_uc_va, c->nvls_bytes);
    d.addrFree((CUdeviceptr)c->nvls_uc_va, c->nvls_bytes);
    CUdevice dev;
    if (d.getDevice(&dev, c->device) == CUDA_SUCCESS) d.mcUnbind(c->nvls_mc, dev, 0, c->nvls_bytes);
    d.memRelease(c->nvls_mem);
  }
  if (c->nvls_mc) drv().memRelease(c->nvls_mc);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_last) cudaEventDestroy(c->ev_last);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (int r = 0; r < FC_MAXR; ++r)
    if (c->own[r]) cudaFree(c->ws[r]);
  delete c;
  return FC_SUCCESS;
}

const char* fc_last_error(const fc_comm_t* c) { return c ? c->err.c_str() : "null communicator"; }

int fc_buffer_export_multi(fc_comm_t* c, const void* const* ptrs, size_t bytes, void* handles) {
  if (!c || !ptrs || !handles) return FC_ERR_INVALID_ARG;
  for (int i = 0; i < c->nlocal; ++i) {
    BufBlob b;
    memset(&b, 0, sizeof(b));
    b.magic = kBufMagic;
    b.rank = c->local[i];
    if (!c->virt) {
      FC_CUDA(c, cudaSetDevice(c->device));
      uintptr_t base = 0;
      size_t size = 0;
      unsigned long long id = 0;
      if (!segment_of(ptrs[i], &base, &size, &id))
        return fail(c, FC_ERR_INVALID_ARG, "pointer %p is not device memory", ptrs[i]);
      if ((uintptr_t)ptrs[i] + bytes > base + size)
        return fail(c, FC_ERR_INVALID_ARG, "buffer exceeds its allocation");
      b.offset = (uintptr_t)ptrs[i] - base;  // the buffer within its mapped segment
      b.bytes = size;
      FC_CUDA(c, cudaIpcGetMemHandle(&b.handle, (void*)base));
    }
    char* dst = (char*)handles + (size_t)i * kHandleBytes;
    memset(dst, 0, kHandleBytes);
    memcpy(dst, &b, sizeof(b));
  }
  return FC_SUCCESS;
}

int fc_buffer_export(fc_comm_t* c, const void* ptr, size_t bytes, void* handle) {
  if (c && c->nlocal != 1) return fail(c, FC_ERR_INVALID_ARG, "use fc_buffer_export_multi");
  return fc_buffer_export_multi(c, &ptr, bytes, handle);
}

// Register the allocation holding one output buffer per local rank
// (ptrs[0..nlocal)); `handles` holds one blob per rank of the communicator,
// in rank order.  Remote ranks' segments are opened via IPC; local ranks use
// the pointers passed per call.  Peers must later pass buffers at the same
// offset within their segments (checked on the device by the buffer tag).
int fc_buffer_register_multi(fc_comm_t* c, const void* const* ptrs, size_t bytes,
                             const void* handles) {
  if (!c || !ptrs) return FC_ERR_INVALID_ARG;
  if (c->virt) return FC_SUCCESS;  // all ranks' buffers are local pointers
  if (!handles) return FC_ERR_INVALID_ARG;
  FC_CUDA(c, cudaSetDevice(c->device));
  Reg reg;
  memset(&reg, 0, sizeof(reg));
  size_t size = 0;
  if (!segment_of(ptrs[0], &reg.lo, &size, &reg.buffer_id))
    return fail(c, FC_ERR_INVALID_ARG, "pointer %p is not device memory", ptrs[0]);
  reg.hi = reg.lo + size;
  reg.anchor = (uintptr_t)ptrs[0];
  if ((uintptr_t)ptrs[0] + bytes > reg.hi)
    return fail(c, FC_ERR_INVALID_ARG, "buffer exceeds its allocation");
  for (int r = 0; r < c->nranks; ++r) {
    BufBlob b;
    memcpy(&b, (const char*)handles + (size_t)r * kHandleBytes, sizeof(b));
    if (b.magic != kBufMagic || b.rank != r)
      return fail(c, FC_ERR_INVALID_ARG, "bad buffer handle for rank %d", r);
    if (c->is_local[r]) continue;
    reg.peer_lo[r] = -(long long)b.offset;
    reg.peer_hi[r] = (long long)b.bytes - (long long)b.offset;
    reg.peer_lo[r] = -(long long)b.offset;
    reg.peer_hi[r] = (long long)b.bytes - (long long)b.offset;
    char* base = nullptr;
    int st = open_mapping(c, b.handle, &base);
    if (st) return st;
    reg.peer[r] = base + b.offset;
  }
  reg.seq = ++c->reg_seq;
  for (auto& r : c->regs)
    if (r.lo == reg.lo) {  // same segment (or a stale one at the same address): replace
      r = reg;
      return FC_SUCCESS;
    }
  c->regs.push_back(reg);
  return FC_SUCCESS;
}

int fc_buffer_register(fc_comm_t* c, const void* ptr, size_t bytes, const void* handles) {
  if (c && c->nlocal != 1 && !c->virt)
    return fail(c, FC_ERR_INVALID_ARG, "use fc_buffer_register_multi");
  return fc_buffer_register_multi(c, &ptr, bytes, handles);
}

int fc_buffer_deregister(fc_comm_t* c, const void* ptr) {
  if (!c) return FC_ERR_INVALID_ARG;
  const uintptr_t a = (uintptr_t)ptr;
  for (size_t i = 0; i < c->regs.size(); ++i)
    if (a >= c->regs[i].lo && a < c->regs[i].hi) {
      c->regs.erase(c->regs.begin() + i);
      return FC_SUCCESS;
    }
  return fail(c, FC_ERR_NOT_REGISTERED, "buffer %p was not registered", ptr);
}

int fc_buffer_query(fc_comm_t* c, const void* ptr, size_t bytes, int* registered) {
  if (!c || !registered) return FC_ERR_INVALID_ARG;
  *registered = (c->virt || c->nranks == 1 || find_reg(c, ptr, bytes) != nullptr) ? 1 : 0;
  return FC_SUCCESS;
}

int fc_buffer_count(const fc_comm_t* c) { return c ? (int)c->regs.size() : -1; }

int fc_call_path(fc_comm_t* c, int collective, size_t count, int dtype, int* path) {
  if (!c || !path || collective < 0 || collective > 2) return FC_ERR_INVALID_ARG;
  const void* no_sends[FC_MAXR] = {};  // decide only: run() touches no buffer
  void* no_recvs[FC_MAXR] = {};
  return run(c, collective, no_sends, no_recvs, count, dtype, FC_SUM, nullptr, path);
}

int fc_call_scratch(fc_comm_t* c, int collective, size_t count, int dtype, size_t cap,
                    size_t* bytes) {
  if (!c || !bytes || collective < 0 || collective > 2) return FC_ERR_INVALID_ARG;
  const void* no_sends[FC_MAXR] = {};
  void* no_recvs[FC_MAXR] = {};
  int path = -1;
  long long need = 0;
  const int st = run(c, collective, no_sends, no_recvs, count, dtype, FC_SUM, nullptr, &path,
                     (long long)align_up(cap, 4096), &need);
  *bytes = need > 0 ? align_up((size_t)need, 4096) : 0;
  return st;
}

size_t fc_comm_scratch_bytes(const fc_comm_t* c) { return c ? c->scratch_bytes : 0; }

// Re-allocate every local workspace with `scratch_bytes` per region.  All
// ranks call it together, after every collective that used the old
// workspaces has completed on every rank (the caller synchronises and
// barriers); the communicator then needs fc_comm_export / fc_comm_connect
// again.  Control blocks and flags restart from zero on every rank alike.
int fc_comm_grow(fc_comm_t* c, size_t scratch_bytes) {
  if (!c) return FC_ERR_INVALID_ARG;
  FC_CUDA(c, cudaSetDevice(c->device));
  FC_CUDA(c, cudaDeviceSynchronize());
  for (int r = 0; r < c->nranks; ++r) {
    if (c->is_local[r] || !c->ws[r]) continue;
    for (size_t i = 0; i < c->maps.size(); ++i)
      if (c->maps[i].base == c->ws[r]) {
        cudaIpcCloseMemHandle(c->maps[i].base);
        c->maps.erase(c->maps.begin() + i);
        break;
      }
    c->ws[r] = nullptr;
  }
  for (int r = 0; r < FC_MAXR; ++r)
    if (c->own[r]) {
      cudaFree(c->ws[r]);
      c->ws[r] = nullptr;
      c->own[r] = false;
    }
  setup_layout(c, scratch_bytes);
  for (int i = 0; i < c->nlocal; ++i) {
    const int st = alloc_workspace(c, &c->ws[c->local[i]]);
    if (st) return st;
    c->own[c->local[i]] = true;
  }
  c->have_last = false;
  c->connected = c->virt || c->nranks == 1;
  return FC_SUCCESS;
}

int fc_plan_load(fc_comm_t* c, int coll, const int32_t* t, size_t nwords) {
  if (!c || !t) return FC_ERR_INVALID_ARG;
  if (coll < 0 || coll > 2) return fail(c, FC_ERR_INVALID_ARG, "bad collective %d", coll);
  if (nwords < FC_HEADER_WORDS || t[TH_MAGIC] != FC_TABLE_MAGIC ||
      t[TH_VERSION] != FC_TABLE_VERSION)
    return fail(c, FC_ERR_PLAN, "not a forest plan table (magic/version)");
  const int N = t[TH_NRANKS], k = t[TH_K], ntrees = t[TH_NTREES], ntasks = t[TH_NTASKS];
  if (t[TH_COLLECTIVE] != coll) return fail(c, FC_ERR_PLAN, "table is for collective %d", t[TH_COLLECTIVE]);
  if (N != c->nranks) return fail(c, FC_ERR_PLAN, "table has %d ranks, comm %d", N, c->nranks);
  if (k < 1 || ntrees < 1 || ntrees > kTreeCap || t[TH_TASK_WORDS] != FC_TASK_WORDS)
    return fail(c, FC_ERR_PLAN, "bad table header (k=%d ntrees=%d)", k, ntrees);
  if (t[TH_MAX_SLOTS] > kSlotCap) return fail(c, FC_ERR_PLAN, "too many slots per rank");
  const size_t task0 = FC_HEADER_WORDS + (size_t)N * FC_RANKDESC_WORDS;
  if (nwords != task0 + (size_t)ntasks * FC_TASK_WORDS)
    return fail(c, FC_ERR_PLAN, "table length %zu does not match header", nwords);
  Plan p;
  p.nranks = N;
  p.k = k;
  p.ntrees = ntrees;
  p.max_slot_units = t[TH_MAX_SLOT_UNITS];
  p.max_slots = t[TH_MAX_SLOTS];
  p.max_ag_slot_units = t[TH_MAX_AG_SLOT_UNITS];
  p.max_ag_slots = t[TH_MAX_AG_SLOTS];
  p.flags = t[TH_FLAGS];
  if (p.max_ag_slots > kSlotCap) return fail(c, FC_ERR_PLAN, "too many staging slots per rank");
  // validate every row
  for (int i = 0; i < ntasks; ++i) {
    const int32_t* T = t + task0 + (size_t)i * FC_TASK_WORDS;
    const int kind = T[TW_KIND];
    if (kind < FC_K_AG_ROOT || kind > FC_K_WAIT_AG || T[TW_TREE] < 0 || T[TW_TREE] >= ntrees ||
        T[TW_ROOT] < 0 || T[TW_ROOT] >= N || T[TW_MLO] < 0 || T[TW_MLO] >= T[TW_MHI] ||
        T[TW_MHI] > k || T[TW_N_AG_CHILD] < 0 || T[TW_N_AG_CHILD] >= FC_MAXR ||
        T[TW_N_RS_CHILD] < 0 || T[TW_N_RS_CHILD] >= FC_MAXR)
      return fail(c, FC_ERR_PLAN, "task row %d is malformed", i);
    for (int j = 0; j < T[TW_N_AG_CHILD]; ++j)
      if (T[TW_AG_CHILD + j] < 0 || T[TW_AG_CHILD + j] >= N)
        return fail(c, FC_ERR_PLAN, "task row %d: bad child rank", i);
    for (int j = 0; j < T[TW_N_RS_CHILD]; ++j)
      if (T[TW_RS_CSLOT + j] < 0 || T[TW_RS_CSLOT + j] >= kSlotCap ||
          T[TW_RS_CPREFIX + j] < 0 || T[TW_RS_CPREFIX + j] > p.max_slot_units)
        return fail(c, FC_ERR_PLAN, "task row %d: bad slot", i);
    if (kind == FC_K_RS_FWD &&
        (T[TW_RS_PARENT] < 0 || T[TW_RS_PARENT] >= N || T[TW_RS_PSLOT] < 0 ||
         T[TW_RS_PSLOT] >= kSlotCap))
      return fail(c, FC_ERR_PLAN, "task row %d: bad reduce parent", i);
    if (T[TW_LAG] < 0 || T[TW_LAG] > 64) return fail(c, FC_ERR_PLAN, "task row %d: bad lag", i);
    p.max_mult = std::max(p.max_mult, T[TW_MHI] - T[TW_MLO]);
  }
  for (int r = 0; r < N; ++r) {
    const int32_t* D = t + FC_HEADER_WORDS + (size_t)r * FC_RANKDESC_WORDS;
    if (D[RD_FIRST] < 0 || D[RD_NACTIVE] < 0 || D[RD_NWAIT] < 0 ||
        D[RD_FIRST] + D[RD_NACTIVE] + D[RD_NWAIT] > ntasks)
      return fail(c, FC_ERR_PLAN, "rank descriptor %d out of range", r);
    p.active_total += D[RD_NACTIVE];
  }
  FC_CUDA(c, cudaSetDevice(c->device));
  for (int i = 0; i < c->nlocal; ++i) {
    const int r = c->local[i];
    const int32_t* D = t + FC_HEADER_WORDS + (size_t)r * FC_RANKDESC_WORDS;
    const int rows = std::max(1, D[RD_NACTIVE] + D[RD_NWAIT]);
    p.nact[i] = D[RD_NACTIVE];
    p.nwait[i] = D[RD_NWAIT];
    for (int j = 0; j < D[RD_NACTIVE] + D[RD_NWAIT]; ++j)
      p.lag_max[i] = std::max(p.lag_max[i], t[task0 + (size_t)(D[RD_FIRST] + j) * FC_TASK_WORDS + TW_LAG]);
    cudaError_t e = cudaMalloc((void**)&p.d_tasks[i], (size_t)rows * FC_TASK_WORDS * 4);
    if (e == cudaSuccess && D[RD_NACTIVE] + D[RD_NWAIT] > 0)
      e = cudaMemcpy(p.d_tasks[i], t + task0 + (size_t)D[RD_FIRST] * FC_TASK_WORDS,
                     (size_t)(D[RD_NACTIVE] + D[RD_NWAIT]) * FC_TASK_WORDS * 4,
                     cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      free_plan(c, p);
      return fail(c, FC_ERR_CUDA, "plan upload failed: %s", cudaGetErrorString(e));
    }
  }
  if (coll != FC_ALLGATHER) {
    // one-shot program for the NVLS engine: per tree, the in-tree children of
    // every rank (its RS row's children, ascending) and a post-order
    std::vector<int32_t> os((size_t)ntrees * FC_OS_TREE_WORDS, 0);
    std::vector<int> seen(ntrees, 0);
    for (int r = 0; r < N; ++r) {
      const int32_t* D = t + FC_HEADER_WORDS + (size_t)r * FC_RANKDESC_WORDS;
      for (int j = 0; j < D[RD_NACTIVE] + D[RD_NWAIT]; ++j) {
        const int32_t* T = t + task0 + (size_t)(D[RD_FIRST] + j) * FC_TASK_WORDS;
        const int kind = T[TW_KIND];
        if (kind != FC_K_RS_FWD && kind != FC_K_RS_ROOT && kind != FC_K_AR_ROOT) continue;
        int32_t* o = os.data() + (size_t)T[TW_TREE] * FC_OS_TREE_WORDS;
        o[OS_ROOT] = T[TW_ROOT];
        o[OS_MLO] = T[TW_MLO];
        o[OS_MHI] = T[TW_MHI];
        o[OS_NCH + r] = T[TW_N_RS_CHILD];
        for (int q = 0; q < T[TW_N_RS_CHILD]; ++q) {
          const int ch = T[TW_RS_CHILD + q];
          if (ch < 0 || ch >= N) return free_plan(c, p), fail(c, FC_ERR_PLAN, "task row: bad reduce child");
          o[OS_CH + r * FC_MAXR + q] = ch;
        }
        ++seen[T[TW_TREE]];
      }
    }
    for (int tr = 0; tr < ntrees; ++tr) {
      if (seen[tr] != N) return free_plan(c, p), fail(c, FC_ERR_PLAN, "tree %d: %d of %d reduce rows", tr, seen[tr], N);
      int32_t* o = os.data() + (size_t)tr * FC_OS_TREE_WORDS;
      // iterative post-order from the root
      int stack[FC_MAXR], idx[FC_MAXR], sp = 0, np = 0;
      stack[sp] = o[OS_ROOT];
      idx[sp++] = 0;
      while (sp > 0) {
        const int v = stack[sp - 1];
        if (idx[sp - 1] < o[OS_NCH + v]) {
          const int ch = o[OS_CH + v * FC_MAXR + idx[sp - 1]++];
          if (sp >= FC_MAXR) return free_plan(c, p), fail(c, FC_ERR_PLAN, "tree %d is not a tree", tr);
          stack[sp] = ch;
          idx[sp++] = 0;
        } else {
          if (np >= N) return free_plan(c, p), fail(c, FC_ERR_PLAN, "tree %d is not a tree", tr);
          o[OS_POST + np++] = v;
          --sp;
        }
      }
      if (np != N) return free_plan(c, p), fail(c, FC_ERR_PLAN, "tree %d does not span the ranks", tr);
      o[OS_NPOST] = np;
    }
    cudaError_t e = cudaMalloc((void**)&p.d_os, os.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(p.d_os, os.data(), os.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      free_plan(c, p);
      return fail(c, FC_ERR_CUDA, "plan upload failed: %s", cudaGetErrorString(e));
    }
    p.os_ntrees = ntrees;
  }
  free_plan(c, c->plans[coll]);
  p.loaded = true;
  c->plans[coll] = p;
  return FC_SUCCESS;
}

int fc_allgather_multi(fc_comm_t* c, const void* const* sends, void* const* recvs,
                       size_t sendcount, int dtype, void* stream) {
  return run(c, FC_ALLGATHER, sends, recvs, sendcount, dtype, FC_SUM, stream);
}
int fc_reduce_scatter_multi(fc_comm_t* c, const void* const* sends, void* const* recvs,
                            size_t recvcount, int dtype, int op, void* stream) {
  return run(c, FC_REDUCE_SCATTER, sends, recvs, recvcount, dtype, op, stream);
}
int fc_allreduce_multi(fc_comm_t* c, const void* const* sends, void* const* recvs,
                       size_t count, int dtype, int op, void* stream) {
  return run(c, FC_ALLREDUCE, sends, recvs, count, dtype, op, stream);
}
int fc_allgather(fc_comm_t* c, const void* send, void* recv, size_t sendcount, int dtype,
                 void* stream) {
  if (c && c->nlocal != 1) return fail(c, FC_ERR_INVALID_ARG, "several local ranks: use fc_allgather_multi");
  return run(c, FC_ALLGATHER, &send, &recv, sendcount, dtype, FC_SUM, stream);
}
int fc_reduce_scatter(fc_comm_t* c, const void* send, void* recv, size_t recvcount, int dtype,
                      int op, void* stream) {
  if (c && c->nlocal != 1) return fail(c, FC_ERR_INVALID_ARG, "several local ranks: use the _multi variant");
  return run(c, FC_REDUCE_SCATTER, &send, &recv, recvcount, dtype, op, stream);
}
int fc_allreduce(fc_comm_t* c, const void* send, void* recv, size_t count, int dtype, int op,
                 void* stream) {
  if (c && c->nlocal != 1) return fail(c, FC_ERR_INVALID_ARG, "several local ranks: use the _multi variant");
  return run(c, FC_ALLREDUCE, &send, &recv, count, dtype, op, stream);
}

int fc_comm_set_trace(fc_comm_t* c, void* records, unsigned int* count, unsigned int cap) {
  if (!c) return FC_ERR_INVALID_ARG;
  if (records && !count) return fail(c, FC_ERR_INVALID_ARG, "trace needs a counter");
  c->trace = (FcTraceRec*)records;
  c->trace_count = records ? count : nullptr;
  c->trace_cap = records ? cap : 0;
  return FC_SUCCESS;
}

int fc_last_call_info(const fc_comm_t* c, long long* info, int ninfo) {
  if (!c || !info) return FC_ERR_INVALID_ARG;
  for (int i = 0; i < ninfo && i < 8; ++i) info[i] = c->info[i];
  return FC_SUCCESS;
}

int fc_nvls_supported(int device) {
  const Drv& d = drv();
  if (!d.ok) return 0;
  CUdevice dev;
  int v = 0;
  if (d.getDevice(&dev, device) != CUDA_SUCCESS) return 0;
  if (d.getAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return 0;
  return v;
}

int fc_nvls_create(fc_comm_t* c, size_t bytes, void* handle) {
  if (!c || !handle || c->virt) return FC_ERR_INVALID_ARG;
  const Drv& d = drv();
  if (!d.ok) return fail(c, FC_ERR_UNSUPPORTED, "driver multicast entry points unavailable");
  FC_CUDA(c, cudaSetDevice(c->device));
  CUmulticastObjectProp prop = mc_prop(c, bytes);
  size_t gran = 0;
  FC_DRV(c, d.mcGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  bytes = (bytes + gran - 1) / gran * gran;
  prop.size = bytes;
  CUmemGenericAllocationHandle mc;
  FC_DRV(c, d.mcCreate(&mc, &prop));
  NvlsBlob blob;
  memset(&blob, 0, sizeof(blob));
  blob.magic = kNvlsMagic;
  blob.bytes = bytes;
  int fd = -1;
  FC_DRV(c, d.exportHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  blob.fd = fd;
  c->nvls_mc = mc;
  c->nvls_bytes = bytes;
  memset(handle, 0, kHandleBytes);
  memcpy(handle, &blob, sizeof(blob));
  return FC_SUCCESS;
}

int fc_nvls_attach(fc_comm_t* c, const void* handle) {
  if (!c || !handle || c->virt) return FC_ERR_INVALID_ARG;
  const Drv& d = drv();
  if (!d.ok) return fail(c, FC_ERR_UNSUPPORTED, "driver multicast entry points unavailable");
  FC_CUDA(c, cudaSetDevice(c->device));
  NvlsBlob blob;
  memcpy(&blob, handle, sizeof(blob));
  if (blob.magic != kNvlsMagic) return fail(c, FC_ERR_INVALID_ARG, "bad NVLS handle");
  if (!c->nvls_mc) {
    CUmemGenericAllocationHandle mc;
    FC_DRV(c, d.importHandle(&mc, (void*)(uintptr_t)blob.fd,
                             CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    c->nvls_mc = mc;
    c->nvls_bytes = blob.bytes;
  }
  CUdevice dev;
  FC_DRV(c, d.getDevice(&dev, c->device));
  FC_DRV(c, d.mcAddDevice(c->nvls_mc, dev));
  return FC_SUCCESS;
}

// After every rank attached (caller barrier): bind local memory, map the
// multicast and unicast views.  Returns the unicast base (the pool).
int fc_nvls_bind(fc_comm_t* c, void** pool) {
  if (!c || !pool || !c->nvls_mc) return FC_ERR_INVALID_ARG;
  const Drv& d = drv();
  FC_CUDA(c, cudaSetDevice(c->device));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mem;
  FC_DRV(c, d.memCreate(&mem, c->nvls_bytes, &ap, 0));
  c->nvls_mem = mem;
  FC_DRV(c, d.mcBindMem(c->nvls_mc, 0, mem, 0, c->nvls_bytes, 0));
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mcva = 0;
  FC_DRV(c, d.addrReserve(&uc, c->nvls_bytes, 0, 0, 0));
  FC_DRV(c, d.memMap(uc, c->nvls_bytes, 0, mem, 0));
  FC_DRV(c, d.setAccess(uc, c->nvls_bytes, &acc, 1));
  FC_DRV(c, d.addrReserve(&mcva, c->nvls_bytes, 0, 0, 0));
  FC_DRV(c, d.memMap(mcva, c->nvls_bytes, 0, c->nvls_mc, 0));
  FC_DRV(c, d.setAccess(mcva, c->nvls_bytes, &acc, 1));
  c->nvls_uc_va = (char*)uc;
  c->nvls_mc_va = (char*)mcva;
  // LL multicast staging: two halves at the top of the pool (allgather <= nvls_ll_max)
  c->nvls_ll_half = (long long)(std::min<size_t>(c->nvls_bytes / 8, 16u << 20) / 4096 * 4096);
  FC_CUDA(c, cudaMemset(c->nvls_uc_va, 0, c->nvls_bytes));
  FC_CUDA(c, cudaDeviceSynchronize());
  c->nvls_bound = 1;
  *pool = c->nvls_uc_va;
  return FC_SUCCESS;
}

int fc_nvls_allgather(fc_comm_t* c, const void* send, void* recv, size_t sendcount, int dtype,
                      void* stream) {
  return run_nvls(c, 0, send, recv, nullptr, sendcount, dtype, FC_SUM, stream);
}
int fc_nvls_reduce_scatter(fc_comm_t* c, const void* send, void* recv, size_t recvcount,
                           int dtype, int op, void* stream) {
  return run_nvls(c, 1, nullptr, (void*)send, recv, recvcount, dtype, op, stream);
}
int fc_nvls_allreduce(fc_comm_t* c, void* buf, size_t count, int dtype, int op, void* stream) {
  return run_nvls(c, 2, nullptr, buf, nullptr, count, dtype, op, stream);
}

}  // extern "C"
