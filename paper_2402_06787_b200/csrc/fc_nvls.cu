// NVLS engine: the ForestColl forest on one multicast/aggregation-capable
// NVSwitch, executed with multimem instructions.
//
// With the switch flagged multicast/aggregation, the reference prunes every
// tree down to one send per root into the switch (prune_multicast /
// prune_aggregation, pkg/src/collsched/schedule.py:237-306; "each GPU then
// sends 1 unit into nvs instead of 7").  Executing the
// pruned forest therefore means:
//   allgather:      root r stores shard r once to the multicast address
//                   (multimem.st) and the switch replicates it to every GPU;
//   reduce-scatter: root r reads shard r once through the switch with
//                   in-network aggregation (multimem.ld_reduce);
//   allreduce:      both, on the same shard.
// Buffers live in a symmetric pool bound to a CUDA multicast object.
// In-switch fp reductions use the switch's accumulation order (fp32
// accumulate for bf16/fp16), so fp results match the tree oracle only within
// tolerance; int32 sums are exact.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "fc_arith.cuh"
#include "fc_internal.h"

#define FC_NVLS_THREADS 512

namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ bool wait_peers(const FcNvlsParams& P, int base, unsigned e) {
  const unsigned* f = P.flags[P.rank] + P.bar_off + base;
  const unsigned long long t0 = globaltimer();
  for (int p = 0; p < P.nranks; ++p) {
    if (p == P.rank) continue;
    while ((int)(ld_acquire_sys(f + p) - e) < 0) {
      if ((long long)(globaltimer() - t0) > P.timeout_ns) {
        atomicCAS(&P.ctl->error, 0u, (unsigned)FC_DEVERR_TIMEOUT_READY);
        return false;
      }
    }
  }
  return true;
}

__device__ __forceinline__ void mm_st(char* p, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "f"(__uint_as_float(v.x)), "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)),
               "f"(__uint_as_float(v.w))
               : "memory");
}

template <int DT>
__device__ __forceinline__ uint4 mm_ld_reduce(const char* p) {
  uint4 r;
  if constexpr (DT == FC_FLOAT32) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "l"(p)
                 : "memory");
    r = make_uint4(__float_as_uint(a), __float_as_uint(b), __float_as_uint(c), __float_as_uint(d));
  } else if constexpr (DT == FC_BFLOAT16) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
  } else if constexpr (DT == FC_FLOAT16) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
  } else {  // int32 / uint32: wrapping add, scalar multimem ops
    const unsigned* q = reinterpret_cast<const unsigned*>(p);
    unsigned v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];"
                   : "=r"(v[i])
                   : "l"(q + i)
                   : "memory");
    r = make_uint4(v[0], v[1], v[2], v[3]);
  }
  return r;
}

// AVG on the NVLS path: the switch's sum (already in the buffer dtype) is
// multiplied by the fp32 1/N and rounded again (NVLS fp results are compared
// within tolerance, see the header comment).
template <int DT>
__device__ __forceinline__ void scale16(uint4& v, float s) {
  unsigned* w = reinterpret_cast<unsigned*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (DT == FC_FLOAT32) {
      w[i] = __float_as_uint(__fmul_rn(__uint_as_float(w[i]), s));
    } else if constexpr (DT == FC_BFLOAT16) {
      __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&w[i]);
      float2 f = __bfloat1622float2(h);
      h = __floats2bfloat162_rn(__fmul_rn(f.x, s), __fmul_rn(f.y, s));
      w[i] = *reinterpret_cast<unsigned*>(&h);
    } else if constexpr (DT == FC_FLOAT16) {
      __half2 h = *reinterpret_cast<__half2*>(&w[i]);
      float2 f = __half22float2(h);
      h = __floats2half2_rn(__fmul_rn(f.x, s), __fmul_rn(f.y, s));
      w[i] = *reinterpret_cast<unsigned*>(&h);
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(FC_NVLS_THREADS) fc_nvls_kernel(const __grid_constant__ FcNvlsParams P) {
  __shared__ unsigned s_e;
  __shared__ int s_ok;
  FcCtl* ctl = P.ctl;
  if (threadIdx.x == 0) {
    s_e = *reinterpret_cast<volatile unsigned*>(&ctl->epoch) + 1;
  }
  __syncthreads();
  const unsigned e = s_e;
  // entry barrier: peers' inputs are ready and their outputs may be written
  if (blockIdx.x == 0 && (int)threadIdx.x < P.nranks && (int)threadIdx.x != P.rank)
    st_release_sys(P.flags[threadIdx.x] + P.bar_off + P.rank, e);
  if (threadIdx.x == 0) s_ok = wait_peers(P, 0, e) ? 1 : 0;
  __syncthreads();
  if (s_ok) {
    const long long r0 = (long long)P.rank * P.shard_bytes;
    long long len = P.total_bytes - r0;
    len = len < 0 ? 0 : (len > P.shard_bytes ? P.shard_bytes : len);
    const long long nv = len / 16;
    const long long stride = (long long)gridDim.x * blockDim.x;
    constexpr int U = 8;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride * U) {
      uint4 v[U];
      if (P.mode == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i + u * stride < nv) v[u] = __ldcg(reinterpret_cast<const uint4*>(P.send) + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i + u * stride < nv) mm_st(P.mc + r0 + 16 * (i + u * stride), v[u]);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i + u * stride < nv) v[u] = mm_ld_reduce<DT>(P.mc + r0 + 16 * (i + u * stride));
        if (P.op == FC_AVG) {
#pragma unroll
          for (int u = 0; u < U; ++u) scale16<DT>(v[u], P.scale);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (i + u * stride >= nv) continue;
          if (P.mode == 1)
            reinterpret_cast<uint4*>(P.out)[i + u * stride] = v[u];
          else
            mm_st(P.mc + r0 + 16 * (i + u * stride), v[u]);
        }
      }
    }
  }
  asm volatile("fence.proxy.alias;" ::: "memory");
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&ctl->done, 1u);
    if (prev == gridDim.x - 1) {
      // exit barrier: every peer finished writing into / reading from this GPU
      for (int t = 0; t < P.nranks; ++t)
        if (t != P.rank) st_release_sys(P.flags[t] + P.bar_off + FC_MAXR + P.rank, e);
      wait_peers(P, FC_MAXR, e);
      asm volatile("fence.proxy.alias;" ::: "memory");
      ctl->done = 0;
      __threadfence();
      atomicExch(&ctl->epoch, e);
    }
  }
}

// Allgather of the multicast-pruned forest with an LL protocol: every root
// stores its shard once into the switch as 16-byte units {d0, e, d1, e} (each
// 8-byte half pairs data with the launch epoch, NCCL's LL idea); the switch
// replicates it into every GPU's staging, and receivers poll their local copy
// until both flags read e.  No entry or exit barrier: staging alternates
// between two halves by epoch parity (a rank in launch e has finished e-1,
// which needed every rank's shard, so every rank has finished e-2, the last
// user of this half).  Output and input may be any device buffers (any
// alignment: ld_u64_any / st_u64_any).
__global__ void __launch_bounds__(FC_NVLS_THREADS) fc_nvls_ll_ag_kernel(const __grid_constant__ FcNvlsParams P) {
  __shared__ unsigned s_e;
  FcCtl* ctl = P.ctl;
  if (threadIdx.x == 0) s_e = *reinterpret_cast<volatile unsigned*>(&ctl->epoch) + 1;
  __syncthreads();
  const unsigned e = s_e;
  const long long half = (long long)(e & 1u) * P.ll_half;
  const long long slot = 2 * P.shard_bytes;  // staging bytes per root
  const long long nunits = P.shard_bytes / 8;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // 1. own shard: one multicast store per 8 payload bytes; local copy direct
  char* own = P.out + (long long)P.rank * P.shard_bytes;
  char* mst = P.mc_stage + half + (long long)P.rank * slot;
  for (long long i = tid; i < nunits; i += stride) {
    const unsigned long long v = ld_u64_any(P.send + 8 * i);
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mst + 16 * i),
                 "f"(__uint_as_float((unsigned)v)), "f"(__uint_as_float(e)),
                 "f"(__uint_as_float((unsigned)(v >> 32))), "f"(__uint_as_float(e))
                 : "memory");
    st_u64_any(own + 8 * i, v);
  }
  // 2. every other root's shard from the local staging copy, root by root
  //    (measured ~1 us faster than gathering all roots' units together)
  const unsigned long long t0 = globaltimer();
  bool ok = true;
  for (int q = 0; q < P.nranks && ok; ++q) {
    if (q == P.rank) continue;
    const char* us = P.uc_stage + half + (long long)q * slot;
    char* dst = P.out + (long long)q * P.shard_bytes;
    for (long long i = tid; i < nunits && ok; i += stride) {
      unsigned a, fa, b, fb;
      for (unsigned it = 0;; ++it) {
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(fa), "=r"(b), "=r"(fb)
                     : "l"(us + 16 * i)
                     : "memory");
        if (fa == e && fb == e) break;
        if ((it & 1023u) == 1023u &&
            (*reinterpret_cast<volatile unsigned*>(&ctl->error) != 0 ||
             (long long)(globaltimer() - t0) > P.timeout_ns)) {
          atomicCAS(&ctl->error, 0u, (unsigned)FC_DEVERR_TIMEOUT_AG);
          ok = false;
          break;
        }
      }
      if (ok) st_u64_any(dst + 8 * i, (unsigned long long)a | ((unsigned long long)b << 32));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&ctl->done, 1u);
    if (prev == gridDim.x - 1) {
      ctl->done = 0;
      atomicExch(&ctl->epoch, e);
    }
  }
}

// The in-tree (one-shot program row) of root r0 whose slice holds elements
// [o0, o1] of that root's shard of Sr elements, or null if they straddle a
// slice boundary (or lie past the shard: allreduce padding).
__device__ __forceinline__ const int* os_tree_of(const FcNvlsParams& P, long long r0,
                                                 long long o0, long long o1, long long Sr) {
  for (int ti = 0; ti < P.os_ntrees && o1 < Sr; ++ti) {
    const int* c = P.os_trees + (long long)ti * FC_OS_TREE_WORDS;
    if (__ldg(c + OS_ROOT) != (int)r0) continue;
    const long long lo = Sr * __ldg(c + OS_MLO) / P.k, hi = Sr * __ldg(c + OS_MHI) / P.k;
    if (o0 >= lo && o1 < hi) return c;
  }
  return nullptr;
}

// Reduce one 8-byte payload word (EPU elements at byte offset `pb` of every
// rank's input; xs[q] = rank q's word) over the forest's in-tree that covers
// it, in the executor's order: post-order; a node adds its own value and its
// children's partials in ascending rank order in the accumulation type and
// rounds once (leaves forward their own value; AVG scales at the root).
// `rs` (reduce-scatter): offsets are relative to `rank`'s shard.  Shared by
// the one-shot kernels; bit-identical to the forest kernel and the oracle.
template <int DT>
__device__ unsigned long long tree_word(const FcNvlsParams& P, bool rs, int rank, long long pb,
                                        const unsigned long long* xs) {
  using R = Red<DT>;
  using E = typename R::E;
  using Acc = typename R::A;
  constexpr int EPU = 8 / (int)sizeof(E);
  const long long S = P.shard_elems;
  const long long g0 = pb / (long long)sizeof(E);
  const int* T0;
  {
    long long r0, o0, Sr;
    if (rs) {
      r0 = rank;
      o0 = g0 - (long long)rank * S;
      Sr = S;
    } else {
      r0 = g0 / S;
      o0 = g0 - r0 * S;
      Sr = P.count - r0 * S;
      Sr = Sr < S ? Sr : S;
    }
    T0 = os_tree_of(P, r0, o0, o0 + EPU - 1, Sr);
  }
  unsigned long long part[FC_MAXR];
  if (T0 != nullptr) {  // the whole word lies in one slice: evaluate all lanes at once
    const int np = __ldg(T0 + OS_NPOST), root = __ldg(T0 + OS_ROOT);
    for (int a = 0; a < np; ++a) {
      const int v = __ldg(T0 + OS_POST + a);
      const int nc = __ldg(T0 + OS_NCH + v);
      if (nc == 0) {
        part[v] = xs[v];
        continue;
      }
      const E* xv = reinterpret_cast<const E*>(&xs[v]);
      Acc acc[EPU];
#pragma unroll
      for (int m = 0; m < EPU; ++m) acc[m] = R::to(xv[m]);
      for (int q = 0; q < nc; ++q) {
        const unsigned long long pc = part[__ldg(T0 + OS_CH + v * FC_MAXR + q)];
        const E* pe = reinterpret_cast<const E*>(&pc);
#pragma unroll
        for (int m = 0; m < EPU; ++m) acc[m] = R::add(acc[m], R::to(pe[m]));
      }
      if (P.op == FC_AVG && v == root) {
#pragma unroll
        for (int m = 0; m < EPU; ++m) acc[m] = R::mul(acc[m], P.scale);
      }
      unsigned long long o;
      E* oe = reinterpret_cast<E*>(&o);
#pragma unroll
      for (int m = 0; m < EPU; ++m) oe[m] = R::from(acc[m]);
      part[v] = o;
    }
    return part[root];
  }
  // a slice boundary inside the word: element by element
  unsigned long long res = 0;
  E* re = reinterpret_cast<E*>(&res);
  for (int m = 0; m < EPU; ++m) {
    const long long gi = g0 + m;
    long long r, o, Sr;
    if (rs) {
      r = rank;
      o = gi - (long long)rank * S;
      Sr = S;
    } else {
      r = gi / S;
      o = gi - r * S;
      Sr = P.count - r * S;
      Sr = Sr < S ? Sr : S;
    }
    const int* T = os_tree_of(P, r, o, o, Sr);
    if (T == nullptr) {  // past the last shard (padding): nothing to reduce
      re[m] = reinterpret_cast<const E*>(&xs[rank])[m];
      continue;
    }
    E pe[FC_MAXR];
    const int np = __ldg(T + OS_NPOST), root = __ldg(T + OS_ROOT);
    for (int a = 0; a < np; ++a) {
      const int v = __ldg(T + OS_POST + a);
      const E xv = reinterpret_cast<const E*>(&xs[v])[m];
      const int nc = __ldg(T + OS_NCH + v);
      if (nc == 0) {
        pe[v] = xv;
        continue;
      }
      Acc acc = R::to(xv);
      for (int q = 0; q < nc; ++q) acc = R::add(acc, R::to(pe[__ldg(T + OS_CH + v * FC_MAXR + q)]));
      if (P.op == FC_AVG && v == root) acc = R::mul(acc, P.scale);
      pe[v] = R::from(acc);
    }
    re[m] = pe[root];
  }
  return res;
}

// Reduce-scatter (mode 4) / allreduce (mode 5) for small buffers on the NVLS
// engine: every rank multicasts its whole input once as LL units (same
// staging scheme as the allgather above), so after one switch hop every GPU
// holds every rank's input.  Each GPU then evaluates the forest's in-trees
// locally in the executor's order (tree_word): bit-identical to the tree
// engine and the oracle.  Allreduce computes the whole buffer on every GPU;
// reduce-scatter only the own shard.  The staging is the pool's own (only
// this 16-byte unit format is ever written there).
template <int DT>
__global__ void __launch_bounds__(FC_NVLS_THREADS) fc_nvls_ll_red_kernel(const __grid_constant__ FcNvlsParams P) {
  __shared__ unsigned s_e;
  FcCtl* ctl = P.ctl;
  if (threadIdx.x == 0) s_e = *reinterpret_cast<volatile unsigned*>(&ctl->epoch) + 1;
  __syncthreads();
  const unsigned e = s_e;
  const long long half = (long long)(e & 1u) * P.ll_half;
  const long long slot = 2 * P.buf_bytes;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const bool rs = P.mode == 4;
  // 1. the whole own input to every rank's staging: one multicast store
  const long long nin = P.buf_bytes / 8;
  char* mst = P.mc_stage + half + (long long)P.rank * slot;
  for (long long i = tid; i < nin; i += stride) {
    const unsigned long long v = ld_u64_any(P.send + 8 * i);
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mst + 16 * i),
                 "f"(__uint_as_float((unsigned)v)), "f"(__uint_as_float(e)),
                 "f"(__uint_as_float((unsigned)(v >> 32))), "f"(__uint_as_float(e))
                 : "memory");
  }
  // 2. output words: allreduce the whole buffer, reduce-scatter the own shard
  using E = typename Red<DT>::E;
  const long long S = P.shard_elems;
  const long long u0 = rs ? (long long)P.rank * S * (long long)sizeof(E) / 8 : 0;
  const long long nout = rs ? S * (long long)sizeof(E) / 8 : nin;
  const unsigned long long t0 = globaltimer();
  for (long long u = tid; u < nout; u += stride) {
    const long long iu = u0 + u;
    unsigned long long x[FC_MAXR];
    // every slot including our own (its arrival proves the input was read),
    // one rank at a time: a single poll in flight per thread keeps the
    // staging reads from competing with the arriving stores
    bool ok = true;
    for (int q = 0; q < P.nranks && ok; ++q) {
      const char* pq = P.uc_stage + half + (long long)q * slot + 16 * iu;
      unsigned a, fa, b, fb;
      for (unsigned it = 0;; ++it) {
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(fa), "=r"(b), "=r"(fb)
                     : "l"(pq)
                     : "memory");
        if (fa == e && fb == e) break;
        if ((it & 1023u) == 1023u &&
            (*reinterpret_cast<volatile unsigned*>(&ctl->error) != 0 ||
             (long long)(globaltimer() - t0) > P.timeout_ns)) {
          atomicCAS(&ctl->error, 0u, (unsigned)FC_DEVERR_TIMEOUT_RS);
          ok = false;
          break;
        }
      }
      x[q] = (unsigned long long)a | ((unsigned long long)b << 32);
    }
    if (!ok) break;
    st_u64_any(P.out + 8 * u, tree_word<DT>(P, rs, P.rank, 8 * iu, x));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&ctl->done, 1u);
    if (prev == gridDim.x - 1) {
      ctl->done = 0;
      atomicExch(&ctl->epoch, e);
    }
  }
}

// The local rank a CTA of a one-shot kernel (modes 6/7/8) serves.  One grid
// runs P.nlocal ranks (one in production; all N in virtual mode, launched
// cooperatively so that ranks of one grid can wait on each other).
struct OneshotView {
  int rank;
  FcCtl* ctl;
  const char* send;
  char* out;
  const char* stage;  // this rank's own staging (peers' lines land here)
  long long cta, nctas;
};

__device__ __forceinline__ OneshotView oneshot_view(const FcNvlsParams& P) {
  OneshotView v;
  const int lr = (int)(blockIdx.x / (unsigned)P.ctas_per_rank);
  v.rank = P.lrank[lr];
  v.ctl = P.lctl[lr];
  v.send = P.lsend[lr];
  v.out = P.lout[lr];
  v.stage = P.peer_stage[v.rank];
  v.cta = blockIdx.x % (unsigned)P.ctas_per_rank;
  v.nctas = P.ctas_per_rank;
  return v;
}

__device__ __forceinline__ void oneshot_finish(const OneshotView& V, const FcNvlsParams& P,
                                               unsigned e) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&V.ctl->done, 1u);
    if (prev == (unsigned)P.ctas_per_rank - 1u) {
      V.ctl->done = 0;
      atomicExch(&V.ctl->epoch, e);
    }
  }
}

// Poll one LL128 line (8-lane group) until its flag (lane 7's second word)
// equals `flag`; warp-uniform.  Returns false on timeout / sticky error.
__device__ __forceinline__ bool poll_line(const char* pq, bool valid, unsigned long long flag,
                                          int lane, unsigned long long& a, unsigned long long& b,
                                          FcCtl* ctl, unsigned long long t0, long long timeout_ns,
                                          unsigned code) {
  const int gl = lane & 7;
  for (unsigned it = 0;; ++it) {
    a = 0;
    b = flag;
    if (valid)
      asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(pq) : "memory");
    const int mine_ok = (!valid || gl != 7 || b == flag) ? 1 : 0;
    const int grp_ok = __shfl_sync(0xffffffffu, mine_ok, (lane & ~7) | 7);
    if (__all_sync(0xffffffffu, grp_ok)) return true;
    if ((it & 1023u) == 1023u) {
      int bad = 0;
      if (lane == 0 && (*reinterpret_cast<volatile unsigned*>(&ctl->error) != 0 ||
                        (long long)(globaltimer() - t0) > timeout_ns)) {
        atomicCAS(&ctl->error, 0u, code);
        bad = 1;
      }
      if (__shfl_sync(0xffffffffu, bad, 0)) return false;
    }
  }
}

// One-shot reduce-scatter (mode 6) / allreduce (mode 7) for the tree engine,
// in LL128 lines: every rank stores its whole input as 128-byte lines (120
// payload bytes + the epoch in the last 8) into every rank's staging through
// the peer mappings -- 1.07x the bytes of the input -- then each GPU
// evaluates the in-trees locally (tree_word).  A warp's 8-lane group moves
// one line; NVLink delivers it whole, so the flag in lane 7 vouches for the
// whole line (the LL128 rule of the forest kernel).  Every writer of the
// tree engine's staging uses this line format, so a flag word there only
// ever holds 0 or an epoch.
template <int DT>
__global__ void __launch_bounds__(FC_NVLS_THREADS) fc_oneshot128_kernel(const __grid_constant__ FcNvlsParams P) {
  using E = typename Red<DT>::E;
  const OneshotView V = oneshot_view(P);
  __shared__ unsigned s_e;
  if (threadIdx.x == 0) s_e = *reinterpret_cast<volatile unsigned*>(&V.ctl->epoch) + 1;
  __syncthreads();
  const unsigned e = s_e;
  const unsigned long long flag = e;
  const bool rs = P.mode == 6;
  const long long B = P.buf_bytes;
  const long long L = (B + 119) / 120;
  const long long slot = L * 128;
  const long long half = (long long)(e & 1u) * P.ll_half;
  const long long mine = half + (long long)V.rank * slot;
  const int lane = threadIdx.x & 31, gl = lane & 7;
  const long long gid = (V.cta * blockDim.x + threadIdx.x) >> 3;  // 8-lane group
  const long long ngrp = (V.nctas * blockDim.x) >> 3;
  const long long p_lane = 16LL * gl;  // this lane's payload bytes within a line: [p_lane, +16)
  // 1. every line of the own input to every rank's staging
  for (long long l = gid; l < L; l += ngrp) {
    const long long pb = 120 * l + p_lane;
    unsigned long long w0 = 0, w1 = flag;
    if (pb + 8 <= B) w0 = ld_u64_any(V.send + pb);
    if (gl < 7) w1 = (pb + 16 <= B) ? ld_u64_any(V.send + pb + 8) : 0ull;
    for (int q = 0; q < P.nranks; ++q)
      asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(P.peer_stage[q] + mine + 128 * l + 16 * gl),
                   "l"(w0), "l"(w1)
                   : "memory");
  }
  // 2. the lines holding output words: all of them (allreduce) or those of the own shard
  const long long S = P.shard_elems;
  const long long ob = rs ? (long long)V.rank * S * (long long)sizeof(E) : 0;  // first output byte
  const long long oe = rs ? ob + S * (long long)sizeof(E) : B;
  const long long l0 = ob / 120, l1 = (oe + 119) / 120;
  const unsigned long long t0 = globaltimer();
  // warp-uniform loop: a warp's 4 groups take 4 consecutive lines per step
  const long long wid = gid >> 2, nw = ngrp >> 2;
  for (long long lb = l0 + 4 * wid; lb < l1; lb += 4 * nw) {
    const long long l = lb + (lane >> 3);
    const bool valid = l < l1;
    unsigned long long x0[FC_MAXR], x1[FC_MAXR];
    bool ok = true;
    for (int q = 0; q < P.nranks && ok; ++q)
      ok = poll_line(V.stage + half + (long long)q * slot + 128 * l + 16 * gl, valid, flag, lane,
                     x0[q], x1[q], V.ctl, t0, P.timeout_ns, FC_DEVERR_TIMEOUT_RS);
    if (!ok) break;
    if (!valid) continue;
    const long long pb = 120 * l + p_lane;
    if (pb >= ob && pb + 8 <= oe) st_u64_any(V.out + (pb - ob), tree_word<DT>(P, rs, V.rank, pb, x0));
    if (gl < 7 && pb + 8 >= ob && pb + 16 <= oe)
      st_u64_any(V.out + (pb + 8 - ob), tree_word<DT>(P, rs, V.rank, pb + 8, x1));
  }
  oneshot_finish(V, P, e);
}

// One-hop allgather (mode 8) for the tree engine's small messages on a
// single-switch forest (FC_PLAN_ONEHOP): every root stores its shard as LL128
// lines straight into every other rank's staging (depth-1 trees: the same
// per-link load as the forest, one hop instead of its depth); receivers copy
// arrived lines to their output.  The own shard is copied locally.  Staging
// halves alternate by epoch parity.
__global__ void __launch_bounds__(FC_NVLS_THREADS) fc_oneshot_ag128_kernel(const __grid_constant__ FcNvlsParams P) {
  const OneshotView V = oneshot_view(P);
  __shared__ unsigned s_e;
  if (threadIdx.x == 0) s_e = *reinterpret_cast<volatile unsigned*>(&V.ctl->epoch) + 1;
  __syncthreads();
  const unsigned e = s_e;
  const unsigned long long flag = e;
  const long long S = P.shard_bytes;
  const long long L = (S + 119) / 120;
  const long long slot = L * 128;
  const long long half = (long long)(e & 1u) * P.ll_half;
  const long long mine = half + (long long)V.rank * slot;
  const int lane = threadIdx.x & 31, gl = lane & 7;
  const long long gid = (V.cta * blockDim.x + threadIdx.x) >> 3;
  const long long ngrp = (V.nctas * blockDim.x) >> 3;
  const long long p_lane = 16LL * gl;
  char* own = V.out + (long long)V.rank * S;
  // 1. own shard: lines to every peer, payload to the own output slot.  The
  // loop is warp-uniform (the warp's 4 line groups step together) so every
  // line leaves as one warp-wide store after __syncwarp.
  for (long long lw = gid & ~3LL; lw < L; lw += ngrp) {
    const long long l = lw + (gid & 3);
    const bool valid = l < L;
    const long long pb = 120 * l + p_lane;
    // a shard whose length is not a multiple of 8 ends in a partial word
    // (zero-padded in the line, stored byte by byte)
    unsigned long long w0 = 0, w1 = flag;
    if (valid) {
      w0 = ld_word(V.send, pb, S);
      st_word(own, pb, S, w0);
      if (gl < 7) {
        w1 = ld_word(V.send, pb + 8, S);
        st_word(own, pb + 8, S, w1);
      }
    }
    __syncwarp();
    if (valid)
      for (int q = 0; q < P.nranks; ++q)
        if (q != V.rank)
          asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(P.peer_stage[q] + mine + 128 * l + 16 * gl),
                       "l"(w0), "l"(w1)
                       : "memory");
  }
  // 2. every other root's lines: warp-uniform, 4 lines per warp step
  const unsigned long long t0 = globaltimer();
  const long long wid = gid >> 2, nw = ngrp >> 2;
  const long long total = (long long)(P.nranks - 1) * L;  // lines to receive
  for (long long jb = 4 * wid; jb < total; jb += 4 * nw) {
    const long long j = jb + (lane >> 3);
    const bool valid = j < total;
    const int qi = valid ? (int)(j / L) : 0;
    const int q = qi < V.rank ? qi : qi + 1;  // skip the own rank
    const long long l = valid ? j - (long long)qi * L : 0;
    unsigned long long a, b;
    if (!poll_line(V.stage + half + (long long)q * slot + 128 * l + 16 * gl, valid, flag, lane, a, b,
                   V.ctl, t0, P.timeout_ns, FC_DEVERR_TIMEOUT_AG))
      break;
    if (!valid) continue;
    char* dst = V.out + (long long)q * S;
    const long long pb = 120 * l + p_lane;
    st_word(dst, pb, S, a);
    if (gl < 7) st_word(dst, pb + 8, S, b);
  }
  oneshot_finish(V, P, e);
}

// A chain in-tree over one 8-byte word, operands in post-order (leaf first):
// the leaf forwards its raw value, every later node adds its own value to
// the partial below and rounds once; AVG scales at the root (the last).
template <int DT, int NR>
__device__ __forceinline__ unsigned long long chain_eval(const FcNvlsParams& P,
                                                         const unsigned long long* x, int n) {
  using R = Red<DT>;
  using E = typename R::E;
  constexpr int EPU = 8 / (int)sizeof(E);
  unsigned long long part = x[0];
#pragma unroll
  for (int i = 1; i < NR; ++i) {
    if (i >= n) break;
    const E* xv = reinterpret_cast<const E*>(&x[i]);
    const E* pv = reinterpret_cast<const E*>(&part);
    unsigned long long o;
    E* oe = reinterpret_cast<E*>(&o);
#pragma unroll
    for (int m = 0; m < EPU; ++m) {
      typename R::A acc = R::add(R::to(xv[m]), R::to(pv[m]));
      if (P.op == FC_AVG && i == n - 1) acc = R::mul(acc, P.scale);
      oe[m] = R::from(acc);
    }
    part = o;
  }
  return part;
}

// Two-hop allreduce (mode 9) / reduce-scatter (mode 10) for mid-size buffers
// on a single-switch forest (FC_PLAN_ONEHOP).  Hop 1: every rank stores its
// input's shard q, as LL128 lines in shard coordinates (line l = shard bytes
// [120 l, 120 l + 120)), into rank q's staging -- (N-1)/N of the input, the
// forest's reduce-scatter load.  Rank q then evaluates shard q over the
// forest's in-tree locally (tree_word: the forest kernel's order, bit-exact)
// and writes it to its output.  Hop 2 (allreduce): it stores the reduced
// lines into every peer's staging, and every rank copies the other roots'
// arrived lines to its output -- the forest's allgather load.  Two hops in
// place of the in-trees' and out-trees' depths; staging halves alternate by
// epoch parity as for every LL128 writer.
template <int DT, int NR>
__global__ void __launch_bounds__(FC_NVLS_THREADS) fc_twohop128_kernel(const __grid_constant__ FcNvlsParams P) {
  using E = typename Red<DT>::E;
  const OneshotView V = oneshot_view(P);
  __shared__ unsigned s_e;
  if (threadIdx.x == 0) s_e = *reinterpret_cast<volatile unsigned*>(&V.ctl->epoch) + 1;
  __syncthreads();
  const unsigned e = s_e;
  const unsigned long long flag = e;
  const bool ar = P.mode == 9;
  const int N = P.nranks, me = V.rank;
  // k = 1 with a chain in-tree (every node at most one child: the
  // single-switch forests): senders are polled in the chain's post-order, so
  // the evaluation below runs in registers, leaf to root
  __shared__ int s_chain[FC_MAXR];
  __shared__ int s_is_chain;
  if (threadIdx.x == 0) {
    s_is_chain = 0;
    if (P.k == 1)
      for (int ti = 0; ti < P.os_ntrees; ++ti) {
        const int* T = P.os_trees + (long long)ti * FC_OS_TREE_WORDS;
        if (__ldg(T + OS_ROOT) != me) continue;
        int chain = __ldg(T + OS_NPOST) == N;
        for (int a = 0; a < N && chain; ++a) {
          const int v = __ldg(T + OS_POST + a);
          s_chain[a] = v;
          chain = __ldg(T + OS_NCH + v) == (a == 0 ? 0 : 1) &&
                  (a == 0 || __ldg(T + OS_CH + v * FC_MAXR) == s_chain[a - 1]);
        }
        s_is_chain = chain;
      }
  }
  __syncthreads();
  const bool is_chain = s_is_chain != 0;
  const long long es = (long long)sizeof(E);
  const long long S = P.shard_elems;
  const long long total = ar ? P.count : S * N;  // elements of the input buffer
  auto shard_bytes = [&](int q) -> long long {
    const long long lo = (long long)q * S, hi = (long long)(q + 1) * S < total ? (long long)(q + 1) * S : total;
    return hi > lo ? (hi - lo) * es : 0;
  };
  const long long Lmax = (S * es + 119) / 120;
  const long long slot = Lmax * 128;
  const long long half = (long long)(e & 1u) * P.ll_half;
  const long long rs_area = half;                           // [sender][line]
  const long long ag_area = half + (long long)N * slot;     // [root][line]
  const int lane = threadIdx.x & 31, gl = lane & 7;
  const long long gid = (V.cta * blockDim.x + threadIdx.x) >> 3;
  const long long ngrp = (V.nctas * blockDim.x) >> 3;
  const long long p_lane = 16LL * gl;
  // hop 1: shard q of the own input -> rank q's staging (the own shard too).
  // Line-major with destinations rotated by the sender's rank: at any moment
  // every rank receives from every sender alike (a destination-major order
  // makes all senders hit one rank's ingress link at a time)
  for (long long j = gid; j < (long long)N * Lmax; j += ngrp) {
    const long long l = j / N;
    const int q = (int)((j - l * N + me) % N);
    const long long Bq = shard_bytes(q);
    if (120 * l >= Bq) continue;
    const char* src = V.send + (long long)q * S * es;
    const long long pb = 120 * l + p_lane;  // shard-relative byte
    unsigned long long w0 = 0, w1 = flag;
    if (pb + 8 <= Bq) w0 = ld_u64_any(src + pb);
    if (gl < 7) w1 = (pb + 16 <= Bq) ? ld_u64_any(src + pb + 8) : 0ull;
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(P.peer_stage[q] + rs_area + (long long)me * slot + 128 * l + 16 * gl),
                 "l"(w0), "l"(w1)
                 : "memory");
  }
  // reduce the own shard as its lines arrive: warp-uniform, 4 lines per warp step
  const unsigned long long t0 = globaltimer();
  const long long wid = gid >> 2, nw = ngrp >> 2;
  const long long Bme = shard_bytes(me);
  const long long Lme = (Bme + 119) / 120;
  const long long base_me = (long long)me * S * es;  // global byte offset of the own shard
  char* out_me = ar ? V.out + base_me : V.out;
  bool ok = true;
  for (long long lb = 4 * wid; lb < Lme && ok; lb += 4 * nw) {
    const long long l = lb + (lane >> 3);
    const bool valid = l < Lme;
    // every sender's line at once: NR loads in flight, one flag check
    unsigned long long x0[FC_MAXR], x1[FC_MAXR];
    unsigned long long c0 = 0, c1 = 0;  // chain: the evaluated words
    for (unsigned it = 0;; ++it) {
      unsigned long long a[NR], b[NR];
      int mine_ok = 1;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        a[q] = 0;
        b[q] = flag;
        const int src = is_chain ? s_chain[q < N ? q : 0] : q;  // chain: post-order
        if (q < N && valid)
          asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                       : "=l"(a[q]), "=l"(b[q])
                       : "l"(V.stage + rs_area + (long long)src * slot + 128 * l + 16 * gl)
                       : "memory");
        mine_ok &= (gl != 7 || b[q] == flag) ? 1 : 0;
      }
      const int grp_ok = __shfl_sync(0xffffffffu, mine_ok, (lane & ~7) | 7);
      if (__all_sync(0xffffffffu, grp_ok)) {
        if (is_chain) {  // leaf to root in registers: one rounding per hop
          c0 = chain_eval<DT, NR>(P, a, N);
          c1 = chain_eval<DT, NR>(P, b, N);
        } else {
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            x0[q] = a[q];
            x1[q] = b[q];
          }
        }
        break;
      }
      if ((it & 1023u) == 1023u) {
        int bad = 0;
        if (lane == 0 && (*reinterpret_cast<volatile unsigned*>(&V.ctl->error) != 0 ||
                          (long long)(globaltimer() - t0) > P.timeout_ns)) {
          atomicCAS(&V.ctl->error, 0u, (unsigned)FC_DEVERR_TIMEOUT_RS);
          bad = 1;
        }
        if (__shfl_sync(0xffffffffu, bad, 0)) {
          ok = false;
          break;
        }
      }
    }
    if (!ok) break;
    const long long pb = 120 * l + p_lane;
    unsigned long long r0 = 0, r1 = gl < 7 ? 0ull : flag;
    if (valid && pb + 8 <= Bme) {
      r0 = is_chain ? c0 : tree_word<DT>(P, !ar, me, base_me + pb, x0);
      st_u64_any(out_me + pb, r0);
    }
    if (valid && gl < 7 && pb + 16 <= Bme) {
      r1 = is_chain ? c1 : tree_word<DT>(P, !ar, me, base_me + pb + 8, x1);
      st_u64_any(out_me + pb + 8, r1);
    }
    if (ar && valid) {  // hop 2: the reduced line to every peer
      for (int q = 0; q < N; ++q)
        if (q != me)
          asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(P.peer_stage[q] + ag_area + (long long)me * slot + 128 * l + 16 * gl),
                       "l"(r0), "l"(r1)
                       : "memory");
    }
  }
  // allreduce: copy the other roots' reduced lines to the output
  if (ar && ok) {
    for (long long jb = 4 * wid; jb < (long long)N * Lmax; jb += 4 * nw) {
      const long long j = jb + (lane >> 3);
      const int q = (int)((j < (long long)N * Lmax ? j : 0) / Lmax);
      const long long l = j - (long long)q * Lmax;
      const long long Bq = shard_bytes(q);
      const bool valid = j < (long long)N * Lmax && q != me && 120 * l < Bq;
      unsigned long long a, b;
      if (!poll_line(V.stage + ag_area + (long long)q * slot + 128 * l + 16 * gl, valid, flag, lane, a,
                     b, V.ctl, t0, P.timeout_ns, FC_DEVERR_TIMEOUT_AG))
        break;
      if (!valid) continue;
      char* dst = V.out + (long long)q * S * es;
      const long long pb = 120 * l + p_lane;
      if (pb + 8 <= Bq) st_u64_any(dst + pb, a);
      if (gl < 7 && pb + 16 <= Bq) st_u64_any(dst + pb + 8, b);
    }
  }
  oneshot_finish(V, P, e);
}

}  // namespace

namespace {
const void* oneshot_fn(int mode, int dtype, int nranks) {
  if (mode == 8) return (const void*)fc_oneshot_ag128_kernel;
  if (mode == 9 || mode == 10) {
#define FC_TWOHOP(NR)                                                             \
  switch (dtype) {                                                                \
    case FC_BFLOAT16: return (const void*)fc_twohop128_kernel<FC_BFLOAT16, NR>;   \
    case FC_FLOAT16: return (const void*)fc_twohop128_kernel<FC_FLOAT16, NR>;     \
    case FC_INT32: return (const void*)fc_twohop128_kernel<FC_INT32, NR>;         \
    default: return (const void*)fc_twohop128_kernel<FC_FLOAT32, NR>;             \
  }
    if (nranks <= 2) FC_TWOHOP(2)
    if (nranks <= 4) FC_TWOHOP(4)
    if (nranks <= 8) FC_TWOHOP(8)
    FC_TWOHOP(16)
#undef FC_TWOHOP
  }
  switch (dtype) {
    case FC_BFLOAT16: return (const void*)fc_oneshot128_kernel<FC_BFLOAT16>;
    case FC_FLOAT16: return (const void*)fc_oneshot128_kernel<FC_FLOAT16>;
    case FC_INT32: return (const void*)fc_oneshot128_kernel<FC_INT32>;
    default: return (const void*)fc_oneshot128_kernel<FC_FLOAT32>;
  }
}
}  // namespace

int fc_oneshot_max_ctas(int mode, int dtype, int nranks, int* out) {
  int per_sm = 0, dev = 0, sms = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, oneshot_fn(mode, dtype, nranks),
                                                                FC_NVLS_THREADS, 0);
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  *out = per_sm * sms;
  return (int)e;
}

int fc_nvls_launch(const FcNvlsParams& p, int ctas, void* stream) {
  void* args[] = {(void*)&p};
  const void* fn;
  if (p.mode == 3)
    return (int)cudaLaunchKernel((const void*)fc_nvls_ll_ag_kernel, dim3(ctas),
                                 dim3(FC_NVLS_THREADS), args, 0, (cudaStream_t)stream);
  if (p.mode >= 6) {
    // tree-engine one-shot: ctas_per_rank CTAs per local rank; ranks of one
    // grid wait on each other, so several local ranks need co-residency
    fn = oneshot_fn(p.mode, p.dtype, p.nranks);
    const dim3 grid(p.nlocal * p.ctas_per_rank);
    if (p.nlocal > 1)
      return (int)cudaLaunchCooperativeKernel(fn, grid, dim3(FC_NVLS_THREADS), args, 0,
                                              (cudaStream_t)stream);
    return (int)cudaLaunchKernel(fn, grid, dim3(FC_NVLS_THREADS), args, 0, (cudaStream_t)stream);
  }
  if (p.mode >= 4) {
    switch (p.dtype) {
      case FC_BFLOAT16: fn = (const void*)fc_nvls_ll_red_kernel<FC_BFLOAT16>; break;
      case FC_FLOAT16: fn = (const void*)fc_nvls_ll_red_kernel<FC_FLOAT16>; break;
      case FC_INT32: fn = (const void*)fc_nvls_ll_red_kernel<FC_INT32>; break;
      default: fn = (const void*)fc_nvls_ll_red_kernel<FC_FLOAT32>; break;
    }
    return (int)cudaLaunchKernel(fn, dim3(ctas), dim3(FC_NVLS_THREADS), args, 0,
                                 (cudaStream_t)stream);
  }
  switch (p.dtype) {
    case FC_BFLOAT16: fn = (const void*)fc_nvls_kernel<FC_BFLOAT16>; break;
    case FC_FLOAT16: fn = (const void*)fc_nvls_kernel<FC_FLOAT16>; break;
    case FC_INT32: fn = (const void*)fc_nvls_kernel<FC_INT32>; break;
    default: fn = (const void*)fc_nvls_kernel<FC_FLOAT32>; break;
  }
  return (int)cudaLaunchKernel(fn, dim3(ctas), dim3(FC_NVLS_THREADS), args, 0,
                               (cudaStream_t)stream);
}
