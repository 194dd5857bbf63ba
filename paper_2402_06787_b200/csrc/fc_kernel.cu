// Persistent sm_100a executor kernel for ForestColl forests.
//
// One grid executes the tree tasks of one or more ranks (one rank per GPU in
// production; all N ranks of a forest on one GPU in virtual mode).  Work is a
// stream of items (task, chunk); workers (groups of FC_WT threads) claim
// items dynamically from a per-rank counter in key order (chunk, stage), so
// every flag wait targets an item with a strictly smaller key and the claim
// order alone guarantees progress.
//
// Data semantics (reference anchors):
//  * allgather: tree (root r, batch j) broadcasts elements
//    [floor(S*lo/k), floor(S*hi/k)) of shard r, lo/hi = cumulative batch
//    multiplicities in schedule order — "a 1/k shard of data is broadcast
//    along each out-tree" (batches: schedule.py:55-59).
//  * reduce-scatter: the same slices travel the reversed in-trees
//    (schedule.py:166-174); a node adds its own slice and its children's
//    partials in ascending rank order, accumulating in fp32 (fp types) or
//    wrapping int32, and rounds to the buffer dtype once per hop.
//  * allreduce: reduce-scatter then allgather on one forest
//    (schedule.py:177-211); the root's reduced chunk is broadcast straight
//    from registers.
// Hops synchronise with system-scope release/acquire flags holding the
// launch epoch; data moves with 16-byte vector loads (L2, .cg) and stores
// issued directly to peer-mapped HBM over NVLink5/NVSwitch.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>

#include "fc_internal.h"

#define FC_WT 128  // threads per worker
#define FC_NW 4    // workers per CTA
#define FC_BLOCK (FC_WT * FC_NW)
#define FC_MAXS 17  // max sources / destinations per item (own + 16)

namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_volatile(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void worker_bar(int w) {
  asm volatile("bar.sync %0, %1;" ::"r"(w + 1), "r"(FC_WT) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *p >= e (wrapping compare).  Returns false on timeout or when
// another worker of this rank already failed.
__device__ bool spin_geq(const unsigned* p, unsigned e, FcCtl* ctl, long long timeout_ns,
                         unsigned code) {
  if ((int)(ld_acquire_sys(p) - e) >= 0) return true;
  const unsigned long long t0 = globaltimer();
  for (unsigned i = 1;; ++i) {
    if ((int)(ld_acquire_sys(p) - e) >= 0) return true;
    if ((i & 1023u) == 0) {
      if (ld_volatile(&ctl->error) != 0) return false;
      if ((long long)(globaltimer() - t0) > timeout_ns) {
        if (atomicCAS(&ctl->error, 0u, code) == 0u) {
          ctl->info[0] = (unsigned)(uintptr_t)p;
          ctl->info[1] = e;
          ctl->info[2] = ld_volatile(p);
        }
        return false;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Element arithmetic.  Accumulation type A; buffer element E.
// ---------------------------------------------------------------------------
template <int DT>
struct Red;

template <>
struct Red<FC_FLOAT32> {
  using E = unsigned;
  using A = float;
  __device__ static A to(E x) { return __uint_as_float(x); }
  __device__ static E from(A a) { return __float_as_uint(a); }
  __device__ static A add(A a, A b) { return __fadd_rn(a, b); }
};

// bf16: fp32 accumulate, one round-to-nearest-even per hop.  NaN is quieted
// the same way as oracle/forest_oracle.py::f32_to_bf16.
template <>
struct Red<FC_BFLOAT16> {
  using E = unsigned short;
  using A = float;
  __device__ static A to(E x) { return __uint_as_float(((unsigned)x) << 16); }
  __device__ static E from(A a) {
    unsigned u = __float_as_uint(a);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (E)((u >> 16) | 0x40u);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (E)(u >> 16);
  }
  __device__ static A add(A a, A b) { return __fadd_rn(a, b); }
};

template <>
struct Red<FC_FLOAT16> {
  using E = unsigned short;
  using A = float;
  __device__ static A to(E x) { return __half2float(__ushort_as_half(x)); }
  __device__ static E from(A a) { return __half_as_ushort(__float2half_rn(a)); }
  __device__ static A add(A a, A b) { return __fadd_rn(a, b); }
};

template <>
struct Red<FC_INT32> {  // also uint32: wrapping two's-complement add
  using E = unsigned;
  using A = unsigned;
  __device__ static A to(E x) { return x; }
  __device__ static E from(A a) { return a; }
  __device__ static A add(A a, A b) { return a + b; }
};

// ---------------------------------------------------------------------------
// Worker-wide data movement.  All pointers of one call share `off`.
// ---------------------------------------------------------------------------
template <typename V, int U>
__device__ __forceinline__ void copy_units(const char* src, char* const* dst, int ndst,
                                           long long off, long long n, int wt) {
  const V* s = reinterpret_cast<const V*>(src + off);
  for (long long i = wt; i < n; i += (long long)FC_WT * U) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + (long long)u * FC_WT;
      if (j < n) v[u] = __ldcg(s + j);
    }
    for (int d = 0; d < ndst; ++d) {
      V* dp = reinterpret_cast<V*>(dst[d] + off);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = i + (long long)u * FC_WT;
        if (j < n) dp[j] = v[u];
      }
    }
  }
}

template <int DT>
__device__ __forceinline__ void reduce_scalar(const char* const* src, int nsrc,
                                              char* const* dst, int ndst, long long off,
                                              long long nelem, int wt) {
  using R = Red<DT>;
  using E = typename R::E;
  for (long long i = wt; i < nelem; i += FC_WT) {
    const long long b = off + i * (long long)sizeof(E);
    typename R::A acc = R::to(__ldcg(reinterpret_cast<const E*>(src[0] + b)));
    for (int s = 1; s < nsrc; ++s)
      acc = R::add(acc, R::to(__ldcg(reinterpret_cast<const E*>(src[s] + b))));
    const E out = R::from(acc);
    for (int d = 0; d < ndst; ++d) *reinterpret_cast<E*>(dst[d] + b) = out;
  }
}

template <int DT, int U>
__device__ __forceinline__ void reduce_vec(const char* const* src, int nsrc, char* const* dst,
                                           int ndst, long long off, long long nvec, int wt) {
  using R = Red<DT>;
  using E = typename R::E;
  using A = typename R::A;
  constexpr int NE = 16 / sizeof(E);
  constexpr int G = 4;  // sources loaded per batch
  for (long long i = wt; i < nvec; i += (long long)FC_WT * U) {
    A acc[U][NE];
    for (int s0 = 0; s0 < nsrc; s0 += G) {
      uint4 x[G][U];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (s0 + g < nsrc) {
          const uint4* sp = reinterpret_cast<const uint4*>(src[s0 + g] + off);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const long long j = i + (long long)u * FC_WT;
            if (j < nvec) x[g][u] = __ldcg(sp + j);
          }
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (s0 + g < nsrc) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const E* e = reinterpret_cast<const E*>(&x[g][u]);
#pragma unroll
            for (int q = 0; q < NE; ++q)
              acc[u][q] = (s0 + g == 0) ? R::to(e[q]) : R::add(acc[u][q], R::to(e[q]));
          }
        }
      }
    }
    uint4 out[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      E* e = reinterpret_cast<E*>(&out[u]);
#pragma unroll
      for (int q = 0; q < NE; ++q) e[q] = R::from(acc[u][q]);
    }
    for (int d = 0; d < ndst; ++d) {
      uint4* dp = reinterpret_cast<uint4*>(dst[d] + off);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = i + (long long)u * FC_WT;
        if (j < nvec) dp[j] = out[u];
      }
    }
  }
}

// Move/reduce nbytes: dst[d][0..n) = reduce(src[0..nsrc))[0..n).  nsrc == 1
// is a pure byte copy (bit-exact for any dtype, NaN payloads included).
template <int DT>
__device__ void xfer(const char* const* src, int nsrc, char* const* dst, int ndst,
                     long long nbytes, int esize, int wt) {
  if (nbytes <= 0 || ndst <= 0) return;
  const uintptr_t a0 = (uintptr_t)src[0];
  uintptr_t diff = 0;
  for (int s = 1; s < nsrc; ++s) diff |= (uintptr_t)src[s] - a0;
  for (int d = 0; d < ndst; ++d) diff |= (uintptr_t)dst[d] - a0;
  if (nsrc == 1) {
    int g = 16;
    while (g > 1 && (diff & (uintptr_t)(g - 1))) g >>= 1;
    long long head = (long long)((g - (a0 & (uintptr_t)(g - 1))) & (uintptr_t)(g - 1));
    if (head > nbytes) head = nbytes;
    for (long long i = wt; i < head; i += FC_WT) {
      const char v = src[0][i];
      for (int d = 0; d < ndst; ++d) dst[d][i] = v;
    }
    const long long nu = (nbytes - head) / g;
    switch (g) {
      case 16: copy_units<uint4, 4>(src[0], dst, ndst, head, nu, wt); break;
      case 8: copy_units<uint2, 4>(src[0], dst, ndst, head, nu, wt); break;
      case 4: copy_units<unsigned, 4>(src[0], dst, ndst, head, nu, wt); break;
      case 2: copy_units<unsigned short, 4>(src[0], dst, ndst, head, nu, wt); break;
      default: copy_units<unsigned char, 4>(src[0], dst, ndst, head, nu, wt); break;
    }
    for (long long i = head + nu * g + wt; i < nbytes; i += FC_WT) {
      const char v = src[0][i];
      for (int d = 0; d < ndst; ++d) dst[d][i] = v;
    }
    return;
  }
  if ((diff & 15) == 0) {
    long long head = (long long)((16 - (a0 & 15)) & 15);
    if (head > nbytes) head = nbytes;
    reduce_scalar<DT>(src, nsrc, dst, ndst, 0, head / esize, wt);
    const long long nv = (nbytes - head) / 16;
    reduce_vec<DT, 2>(src, nsrc, dst, ndst, head, nv, wt);
    const long long t0 = head + nv * 16;
    reduce_scalar<DT>(src, nsrc, dst, ndst, t0, (nbytes - t0) / esize, wt);
  } else {
    reduce_scalar<DT>(src, nsrc, dst, ndst, 0, nbytes / esize, wt);
  }
}

struct Geo {
  long long base, lo, hi;
};

__device__ __forceinline__ long long chunk_bound(const Geo& g, int c, int n) {
  if (c <= 0) return g.lo;
  if (c >= n) return g.hi;
  const long long len = g.hi - g.lo;
  long long b = (g.lo + len * c / n) & ~(long long)(FC_ALIGN - 1);
  return b < g.lo ? g.lo : b;
}

template <int DT>
__device__ void run_item(const FcParams& P, int me, FcCtl* ctl, const int* T, int c,
                         unsigned e, int w, int wt, unsigned& ready_mask, int* s_ok) {
  const int kind = __ldg(T + TW_KIND);
  const int t = __ldg(T + TW_TREE);
  const int root = __ldg(T + TW_ROOT);
  const long long es = P.esize;
  long long Sr = P.total_elems - (long long)root * P.stride_elems;
  Sr = Sr < 0 ? 0 : (Sr > P.shard_elems ? P.shard_elems : Sr);
  Geo g;
  g.base = (long long)root * P.stride_elems * es;
  g.lo = g.base + (Sr * __ldg(T + TW_MLO) / P.k) * es;
  g.hi = g.base + (Sr * __ldg(T + TW_MHI) / P.k) * es;
  const long long b0 = chunk_bound(g, c, P.nchunks);
  const long long b1 = chunk_bound(g, c + 1, P.nchunks);
  const long long wbase = chunk_bound(g, P.c0, P.nchunks) & ~(long long)(FC_ALIGN - 1);
  const int fi = c - P.c0;
  unsigned* const myflags = P.flags[me];
  const int n_ag = __ldg(T + TW_N_AG_CHILD);
  const int n_rs = __ldg(T + TW_N_RS_CHILD);
  const int rs_parent = __ldg(T + TW_RS_PARENT);

  // 1. wait for inputs (parent / children flags) and for destination ranks
  //    to have entered this launch (entry barrier, guards buffer reuse).
  if (wt == 0) {
    bool ok = true;
    if (kind == FC_K_AG_FWD || kind == FC_K_WAIT_AG)
      ok = spin_geq(myflags + P.ag_flag_off + t * P.maxc + fi, e, ctl, P.timeout_ns,
                    FC_DEVERR_TIMEOUT_AG);
    if (kind == FC_K_RS_FWD || kind == FC_K_RS_ROOT || kind == FC_K_AR_ROOT) {
      for (int j = 0; j < n_rs && ok; ++j)
        ok = spin_geq(myflags + P.rs_flag_off + __ldg(T + TW_RS_CSLOT + j) * P.maxc + fi, e,
                      ctl, P.timeout_ns, FC_DEVERR_TIMEOUT_RS);
    }
    if (kind != FC_K_WAIT_AG && kind != FC_K_RS_ROOT) {
      const int nx = (kind == FC_K_RS_FWD) ? 1 : n_ag;
      for (int j = 0; j < nx && ok; ++j) {
        const int x = (kind == FC_K_RS_FWD) ? rs_parent : __ldg(T + TW_AG_CHILD + j);
        if (!((ready_mask >> x) & 1u)) {
          ok = spin_geq(myflags + x, e, ctl, P.timeout_ns, FC_DEVERR_TIMEOUT_READY);
          if (ok) ready_mask |= 1u << x;
        }
      }
    }
    s_ok[w] = ok ? 1 : 0;
  }
  if (kind == FC_K_WAIT_AG) return;
  worker_bar(w);
  if (!s_ok[w]) return;

  // 2. move / reduce the chunk
  const char* src[FC_MAXS];
  char* dst[FC_MAXS];
  int ns = 0, nd = 0;
  const long long slot_phase = b0 - wbase;
  if (kind == FC_K_AG_ROOT || kind == FC_K_AG_FWD) {
    src[ns++] = (kind == FC_K_AG_ROOT) ? P.send[me] + (b0 - g.base) : P.recv[me] + b0;
    if (kind == FC_K_AG_ROOT && P.recv[me] + b0 != src[0]) dst[nd++] = P.recv[me] + b0;
    for (int j = 0; j < n_ag; ++j) dst[nd++] = P.recv[__ldg(T + TW_AG_CHILD + j)] + b0;
  } else {
    src[ns++] = P.send[me] + b0;
    for (int j = 0; j < n_rs; ++j)
      src[ns++] = P.scratch[me] + P.unit_bytes * __ldg(T + TW_RS_CPREFIX + j) +
                  2LL * FC_ALIGN * __ldg(T + TW_RS_CSLOT + j) + slot_phase;
    if (kind == FC_K_RS_FWD) {
      dst[nd++] = P.scratch[rs_parent] + P.unit_bytes * __ldg(T + TW_RS_PPREFIX) +
                  2LL * FC_ALIGN * __ldg(T + TW_RS_PSLOT) + slot_phase;
    } else if (kind == FC_K_RS_ROOT) {
      dst[nd++] = P.recv[me] + (b0 - g.base);
    } else {  // FC_K_AR_ROOT
      dst[nd++] = P.recv[me] + b0;
      for (int j = 0; j < n_ag; ++j) dst[nd++] = P.recv[__ldg(T + TW_AG_CHILD + j)] + b0;
    }
  }
  xfer<DT>(src, ns, dst, nd, b1 - b0, P.esize, wt);

  // 3. publish: make the stores visible system-wide, then release the flags
  if (kind == FC_K_RS_ROOT) return;
  fence_sys();
  worker_bar(w);
  if (wt == 0) {
    if (kind == FC_K_RS_FWD) {
      st_release_sys(P.flags[rs_parent] + P.rs_flag_off + __ldg(T + TW_RS_PSLOT) * P.maxc + fi, e);
    } else {
      for (int j = 0; j < n_ag; ++j)
        st_release_sys(P.flags[__ldg(T + TW_AG_CHILD + j)] + P.ag_flag_off + t * P.maxc + fi, e);
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(FC_BLOCK) fc_forest_kernel(const __grid_constant__ FcParams P) {
  __shared__ int s_item[FC_NW][2];
  __shared__ int s_ok[FC_NW];
  __shared__ unsigned s_epoch;
  const int lr = blockIdx.x / P.ctas_per_rank;
  const int me = P.local_rank[lr];
  FcCtl* const ctl = P.ctl[lr];
  if (threadIdx.x == 0) s_epoch = ld_volatile(&ctl->epoch) + 1;
  __syncthreads();
  const unsigned e = s_epoch;
  // entry barrier: tell every peer that this rank entered launch e
  if ((int)threadIdx.x < P.nranks && (int)threadIdx.x != me)
    st_release_sys(P.flags[threadIdx.x] + me, e);

  const int w = threadIdx.x / FC_WT;
  const int wt = threadIdx.x % FC_WT;
  const int* const tasks = P.tasks[lr];
  const int nact = P.nactive[lr];
  const int nwait = P.nwait[lr];
  const long long W = P.c1 - P.c0;
  const long long nA = (long long)nact * W;
  const long long total = nA + (long long)nwait * W;
  unsigned ready_mask = 1u << me;
  for (int it = 0;; ++it) {
    if (wt == 0) {
      int v = (int)atomicAdd(&ctl->claim, 1u);
      if (ld_volatile(&ctl->error) != 0) v = INT_MAX;
      s_item[w][it & 1] = v;
    }
    worker_bar(w);
    const long long item = s_item[w][it & 1];
    if (item >= total) break;
    int c, ti;
    if (item < nA) {
      c = (int)(item / nact);
      ti = (int)(item - (long long)c * nact);
    } else {
      const long long j = item - nA;
      c = (int)(j / nwait);
      ti = nact + (int)(j - (long long)c * nwait);
    }
    run_item<DT>(P, me, ctl, tasks + (long long)ti * FC_TASK_WORDS, P.c0 + c, e, w, wt,
                 ready_mask, s_ok);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&ctl->done, 1u);
    if (prev == (unsigned)P.ctas_per_rank - 1u) {
      ctl->claim = 0;
      ctl->done = 0;
      __threadfence();
      atomicExch(&ctl->epoch, e);
    }
  }
}

const void* kernel_for(int rd) {
  switch (rd) {
    case FC_BFLOAT16: return (const void*)fc_forest_kernel<FC_BFLOAT16>;
    case FC_FLOAT16: return (const void*)fc_forest_kernel<FC_FLOAT16>;
    case FC_INT32: return (const void*)fc_forest_kernel<FC_INT32>;
    default: return (const void*)fc_forest_kernel<FC_FLOAT32>;
  }
}

}  // namespace

int fc_launch(const FcParams& p, int reduce_dtype, int cooperative, void* stream, int* grid_out) {
  const dim3 grid(p.nlocal * p.ctas_per_rank), block(FC_BLOCK);
  void* args[] = {(void*)&p};
  const void* fn = kernel_for(reduce_dtype);
  if (grid_out) *grid_out = (int)grid.x;
  cudaError_t err;
  if (cooperative)
    err = cudaLaunchCooperativeKernel(fn, grid, block, args, 0, (cudaStream_t)stream);
  else
    err = cudaLaunchKernel(fn, grid, block, args, 0, (cudaStream_t)stream);
  return (int)err;
}

int fc_max_ctas_per_sm(int reduce_dtype, int* out) {
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel_for(reduce_dtype),
                                                           FC_BLOCK, 0);
}
