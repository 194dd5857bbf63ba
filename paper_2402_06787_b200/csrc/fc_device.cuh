#pragma once
// Persistent sm_100a executor kernel for ForestColl forests.
//
// One grid executes the tree tasks of one or more ranks (one rank per GPU in
// production; all N ranks of a forest on one GPU in virtual mode).  Work is a
// stream of items (task, chunk).  Workers — single warps, FC_WPC per CTA,
// each owning an FC_NST-stage shared-memory ring — claim items dynamically
// from a per-rank counter in a skewed key order (chunk + lag*stage, stage):
// every flag wait targets an item with a strictly smaller key, so claim order
// alone guarantees progress, and the lag lets a consumer's
// input usually be complete by the time the item is claimed.
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
//    (schedule.py:177-211); the root's reduced chunk is stored straight to
//    its own buffer and to its broadcast children.
//
// Data movement (Blackwell TMA bulk-copy engine): a worker's lane 0 streams
// its chunk through the smem ring with cp.async.bulk global->shared loads
// (mbarrier complete_tx) and, for copies, cp.async.bulk shared->global stores
// issued once per destination straight into peer-mapped HBM over
// NVLink5/NVSwitch (one local read feeds every child).  Reductions read the
// bulk-loaded sources from smem with all 32 lanes and store 16-byte vectors.
// Hops synchronise with system-scope release/acquire flags holding the
// launch epoch.  Unaligned heads/tails use 16/8/4/2/1-byte vector loops.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <type_traits>

#include "fc_internal.h"
#include "fc_arith.cuh"

#define FC_SMEM_BYTES (FC_WPC * FC_NST * FC_STAGE)

#define FC_WPC 8                           // warps per CTA
// WW (template): warps per worker; a worker holds one item in flight.
#define FC_BLOCK (32 * FC_WPC)
#define FC_NST 3                           // smem stages per worker
#define FC_STAGE (8 * 1024)                // bytes per stage
#define FC_SMEM (FC_WPC * FC_NST * FC_STAGE)
#define FC_MAXS 17                         // max sources / destinations per item
#ifndef FC_RED_U
#define FC_RED_U 2                         // vectors per lane in flight in bulk_reduce
#endif
#ifndef FC_RED_U2
#define FC_RED_U2 1                        // the same for 2-byte types
#endif

namespace {

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_volatile(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// Barrier of one worker (WW warps): a warp barrier or a named CTA barrier
// (id 0 is __syncthreads).
template <int WW>
__device__ __forceinline__ void worker_sync(int wk) {
  if constexpr (WW == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(wk + 1), "r"(WW * 32) : "memory");
  }
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, unsigned bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
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

// Wait until destination rank x has entered launch e.  While x is in launch
// e (it cannot leave it before receiving from us), the output-buffer tag it
// published with its ready epoch must equal ours: a rank that passed a
// differently registered buffer (or offset / size) fails loudly instead of
// receiving stores meant for another buffer.
// The ready slot is one 64-bit word: epoch in the low half, the sender's
// 32-bit tag in the high half, published by one release store.
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned tag32(const FcParams& P) {
  return (unsigned)(P.tag ^ (P.tag >> 32));
}

__device__ bool wait_ready(const FcParams& P, int me, int x, unsigned e, FcCtl* ctl) {
  const unsigned long long* f = reinterpret_cast<const unsigned long long*>(P.flags[me]) + x;
  unsigned long long v = ld_acquire_sys64(f);
  if ((int)((unsigned)v - e) < 0) {
    const unsigned long long t0 = globaltimer();
    for (unsigned i = 1;; ++i) {
      v = ld_acquire_sys64(f);
      if ((int)((unsigned)v - e) >= 0) break;
      if ((i & 1023u) == 0) {
        if (ld_volatile(&ctl->error) != 0) return false;
        if ((long long)(globaltimer() - t0) > P.timeout_ns) {
          if (atomicCAS(&ctl->error, 0u, (unsigned)FC_DEVERR_TIMEOUT_READY) == 0u) {
            ctl->info[0] = (unsigned)x;
            ctl->info[1] = e;
            ctl->info[2] = (unsigned)v;
          }
          return false;
        }
      }
    }
  }
  if ((unsigned)v != e || (unsigned)(v >> 32) == tag32(P)) return true;
  if (atomicCAS(&ctl->error, 0u, (unsigned)FC_DEVERR_BUFFER_MISMATCH) == 0u) {
    ctl->info[0] = (unsigned)x;
    ctl->info[1] = tag32(P);
    ctl->info[2] = (unsigned)(v >> 32);
  }
  return false;
}

// Element q (a compile-time constant after unrolling) of a packed vector in
// the accumulator type.  bf16 unpacks word-wise: the low half shifted up,
// the high half masked in place (one ALU op per element).
template <int DT>
__device__ __forceinline__ typename Red<DT>::A elem(const void* v, int q) {
  if constexpr (DT == FC_BFLOAT16) {
    const unsigned w = reinterpret_cast<const unsigned*>(v)[q >> 1];
    return __uint_as_float((q & 1) ? (w & 0xffff0000u) : (w << 16));
  } else {
    return Red<DT>::to(reinterpret_cast<const typename Red<DT>::E*>(v)[q]);
  }
}

// acc (accumulator lanes of one 16-byte vector) <- first source
template <int DT>
struct Acc16 {
  using R = Red<DT>;
  using E = typename R::E;
  static constexpr int NE = 16 / sizeof(E);
  typename R::A a[NE];
  __device__ __forceinline__ void init(const uint4& v) {
#pragma unroll
    for (int q = 0; q < NE; ++q) a[q] = elem<DT>(&v, q);
  }
  __device__ __forceinline__ void add(const uint4& v) {
#pragma unroll
    for (int q = 0; q < NE; ++q) a[q] = R::add(a[q], elem<DT>(&v, q));
  }
  __device__ __forceinline__ void scale(float s) {
#pragma unroll
    for (int q = 0; q < NE; ++q) a[q] = R::mul(a[q], s);
  }
  __device__ __forceinline__ uint4 pack() const {
    uint4 out;
    if constexpr (sizeof(E) == 2) {
      unsigned* w = reinterpret_cast<unsigned*>(&out);
#pragma unroll
      for (int q = 0; q < NE / 2; ++q) w[q] = R::from2(a[2 * q], a[2 * q + 1]);
    } else {
      E* e = reinterpret_cast<E*>(&out);
#pragma unroll
      for (int q = 0; q < NE; ++q) e[q] = R::from(a[q]);
    }
    return out;
  }
};

// 8-byte (one LL payload word) variant of Acc16.
template <int DT>
struct Acc8 {
  using R = Red<DT>;
  using E = typename R::E;
  static constexpr int NE = 8 / sizeof(E);
  typename R::A a[NE];
  __device__ __forceinline__ void init(unsigned long long v) {
#pragma unroll
    for (int q = 0; q < NE; ++q) a[q] = elem<DT>(&v, q);
  }
  __device__ __forceinline__ void add(unsigned long long v) {
#pragma unroll
    for (int q = 0; q < NE; ++q) a[q] = R::add(a[q], elem<DT>(&v, q));
  }
  __device__ __forceinline__ void scale(float s) {
#pragma unroll
    for (int q = 0; q < NE; ++q) a[q] = R::mul(a[q], s);
  }
  __device__ __forceinline__ unsigned long long pack() const {
    unsigned long long out;
    if constexpr (sizeof(E) == 2) {
      unsigned* w = reinterpret_cast<unsigned*>(&out);
#pragma unroll
      for (int q = 0; q < NE / 2; ++q) w[q] = R::from2(a[2 * q], a[2 * q + 1]);
    } else {
      E* e = reinterpret_cast<E*>(&out);
#pragma unroll
      for (int q = 0; q < NE; ++q) e[q] = R::from(a[q]);
    }
    return out;
  }
};

// ---------------------------------------------------------------------------
// LL128 lines: 120 payload bytes + an 8-byte flag per 128-byte line, written
// by 8 lanes with one 16-byte store each (lane 7 carries the flag).  NVLink
// delivers a warp's 128-byte line store whole, so a reader that sees the
// flag sees the payload: no fence, no separate flag, per-line cut-through.
// ---------------------------------------------------------------------------
#define FC_LL_PAY 120
__device__ __forceinline__ void st_line16(char* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_line16(const char* p, unsigned long long& a,
                                          unsigned long long& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// ---------------------------------------------------------------------------
// Warp-level fallback movers (unaligned / heads / tails).  All pointers of
// one call share `off`.
// ---------------------------------------------------------------------------
template <typename V, int U>
__device__ __forceinline__ void warp_copy_units(const char* src, char* const* dst, int ndst,
                                                long long off, long long n, int lane) {
  const V* s = reinterpret_cast<const V*>(src + off);
  for (long long i = lane; i < n; i += 32LL * U) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + 32LL * u;
      if (j < n) v[u] = __ldcg(s + j);
    }
    for (int d = 0; d < ndst; ++d) {
      V* dp = reinterpret_cast<V*>(dst[d] + off);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = i + 32LL * u;
        if (j < n) dp[j] = v[u];
      }
    }
  }
}

__device__ void warp_copy(const char* src, char* const* dst, int ndst, long long off,
                          long long nbytes, int lane) {
  if (nbytes <= 0) return;
  const uintptr_t a0 = (uintptr_t)src + off;
  uintptr_t diff = 0;
  for (int d = 0; d < ndst; ++d) diff |= (uintptr_t)dst[d] - (uintptr_t)src;
  int g = 16;
  while (g > 1 && (diff & (uintptr_t)(g - 1))) g >>= 1;
  long long head = (long long)((g - (a0 & (uintptr_t)(g - 1))) & (uintptr_t)(g - 1));
  if (head > nbytes) head = nbytes;
  for (long long i = lane; i < head; i += 32) {
    const char v = src[off + i];
    for (int d = 0; d < ndst; ++d) dst[d][off + i] = v;
  }
  const long long nu = (nbytes - head) / g;
  const long long o2 = off + head;
  switch (g) {
    case 16: warp_copy_units<uint4, 4>(src, dst, ndst, o2, nu, lane); break;
    case 8: warp_copy_units<uint2, 4>(src, dst, ndst, o2, nu, lane); break;
    case 4: warp_copy_units<unsigned, 8>(src, dst, ndst, o2, nu, lane); break;
    case 2: warp_copy_units<unsigned short, 8>(src, dst, ndst, o2, nu, lane); break;
    default: warp_copy_units<unsigned char, 8>(src, dst, ndst, o2, nu, lane); break;
  }
  for (long long i = head + nu * g + lane; i < nbytes; i += 32) {
    const char v = src[off + i];
    for (int d = 0; d < ndst; ++d) dst[d][off + i] = v;
  }
}

template <int DT, bool SC>
__device__ void warp_reduce_scalar(const char* const* src, int nsrc, char* const* dst, int ndst,
                                   long long off, long long nelem, int lane, bool scaled, float sc) {
  using R = Red<DT>;
  using E = typename R::E;
  for (long long i = lane; i < nelem; i += 32) {
    const long long b = off + i * (long long)sizeof(E);
    typename R::A acc = R::to(__ldcg(reinterpret_cast<const E*>(src[0] + b)));
    for (int s = 1; s < nsrc; ++s)
      acc = R::add(acc, R::to(__ldcg(reinterpret_cast<const E*>(src[s] + b))));
    if constexpr (SC) {
      if (scaled) acc = R::mul(acc, sc);
    }
    const E out = R::from(acc);
    for (int d = 0; d < ndst; ++d) *reinterpret_cast<E*>(dst[d] + b) = out;
  }
}

template <int DT, bool SC>
__device__ void warp_reduce_vec(const char* const* src, int nsrc, char* const* dst, int ndst,
                                long long off, long long nvec, int lane, bool scaled, float sc) {
  for (long long i = lane; i < nvec; i += 32) {
    Acc16<DT> acc;
    acc.init(__ldcg(reinterpret_cast<const uint4*>(src[0] + off) + i));
    for (int s = 1; s < nsrc; ++s) acc.add(__ldcg(reinterpret_cast<const uint4*>(src[s] + off) + i));
    if constexpr (SC) {
      if (scaled) acc.scale(sc);
    }
    const uint4 out = acc.pack();
    for (int d = 0; d < ndst; ++d) reinterpret_cast<uint4*>(dst[d] + off)[i] = out;
  }
}

// ---------------------------------------------------------------------------
// Per-worker bulk (TMA) movers.  `seq` counts stage fills issued by this
// worker (uniform across its lanes) and selects stage / mbarrier parity.
// ---------------------------------------------------------------------------
struct Ring {
  char* buf;      // FC_NST * FC_STAGE bytes
  uint64_t* bar;  // FC_NST mbarriers
  unsigned seq;
};

// Copy `nbytes` (16-aligned src/dst, multiple of 16) from src + off0 to
// every dst[d] + off0.  Lane 0 issues; bulk store groups stay pending (caller
// waits before flags).  Pointer arrays live in shared memory (no local-memory
// copies on any mover path).
__device__ void bulk_copy(Ring& rg, const char* src, char* const* dst, int ndst, long long off0,
                          long long nbytes, int lane) {
  src += off0;
  const long long npieces = (nbytes + FC_STAGE - 1) / FC_STAGE;
  if (lane == 0) {
    const unsigned base = rg.seq;
    for (long long i = 0; i < npieces && i < FC_NST - 1; ++i) {
      const unsigned q = base + (unsigned)i;
      const long long off = i * FC_STAGE;
      const unsigned len = (unsigned)((nbytes - off) < FC_STAGE ? (nbytes - off) : FC_STAGE);
      mbar_expect_tx(&rg.bar[q % FC_NST], len);
      bulk_load(rg.buf + (q % FC_NST) * FC_STAGE, src + off, len, &rg.bar[q % FC_NST]);
    }
    for (long long i = 0; i < npieces; ++i) {
      const unsigned q = base + (unsigned)i;
      mbar_wait(&rg.bar[q % FC_NST], (q / FC_NST) & 1u);
      const char* sb = rg.buf + (q % FC_NST) * FC_STAGE;
      const long long off = i * FC_STAGE;
      const unsigned len = (unsigned)((nbytes - off) < FC_STAGE ? (nbytes - off) : FC_STAGE);
      for (int d = 0; d < ndst; ++d) bulk_store(dst[d] + off0 + off, sb, len);
      bulk_commit();
      const long long nx = i + FC_NST - 1;
      if (nx < npieces) {
        bulk_wait_read1();  // the stage of piece i-1 (== nx's stage) has been read out
        const unsigned q2 = base + (unsigned)nx;
        const long long off2 = nx * FC_STAGE;
        const unsigned len2 = (unsigned)((nbytes - off2) < FC_STAGE ? (nbytes - off2) : FC_STAGE);
        mbar_expect_tx(&rg.bar[q2 % FC_NST], len2);
        bulk_load(rg.buf + (q2 % FC_NST) * FC_STAGE, src + off2, len2, &rg.bar[q2 % FC_NST]);
      }
    }
  }
  rg.seq += (unsigned)npieces;
}

// Copy with bulk (TMA) loads into the ring and 16-byte lane stores to every
// destination: smem is released as soon as the lanes have read a stage, so
// outstanding NVLink writes hold no shared memory.
__device__ void bulk_copy_stg(Ring& rg, const char* src, char* const* dst, int ndst,
                              long long off0, long long nbytes, int lane) {
  src += off0;
  const long long npieces = (nbytes + FC_STAGE - 1) / FC_STAGE;
  const unsigned base = rg.seq;
  if (lane == 0) {
    for (long long i = 0; i < npieces && i < FC_NST - 1; ++i) {
      const unsigned q = base + (unsigned)i;
      const long long off = i * FC_STAGE;
      const unsigned len = (unsigned)((nbytes - off) < FC_STAGE ? (nbytes - off) : FC_STAGE);
      mbar_expect_tx(&rg.bar[q % FC_NST], len);
      bulk_load(rg.buf + (q % FC_NST) * FC_STAGE, src + off, len, &rg.bar[q % FC_NST]);
    }
  }
  for (long long i = 0; i < npieces; ++i) {
    const unsigned q = base + (unsigned)i;
    mbar_wait(&rg.bar[q % FC_NST], (q / FC_NST) & 1u);
    const uint4* sb = reinterpret_cast<const uint4*>(rg.buf + (q % FC_NST) * FC_STAGE);
    const long long off = i * FC_STAGE;
    const int nv = (int)(((nbytes - off) < FC_STAGE ? (nbytes - off) : FC_STAGE) / 16);
    // the stage in halves: 8 vectors per lane in registers (a full stage
    // would hold 16, pushing the kernel past 255 registers)
    constexpr int PER = FC_STAGE / 16 / 32 / 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint4 v[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int j = lane + 32 * (u + PER * h);
        if (j < nv) v[u] = sb[j];
      }
      if (h == 1) {
        __syncwarp();  // every lane has read the stage: refill it
        if (lane == 0 && i + FC_NST - 1 < npieces) {
          const long long p = i + FC_NST - 1;
          const unsigned q2 = base + (unsigned)p;
          const long long off2 = p * FC_STAGE;
          const unsigned len2 = (unsigned)((nbytes - off2) < FC_STAGE ? (nbytes - off2) : FC_STAGE);
          fence_proxy_async_smem();
          mbar_expect_tx(&rg.bar[q2 % FC_NST], len2);
          bulk_load(rg.buf + (q2 % FC_NST) * FC_STAGE, src + off2, len2, &rg.bar[q2 % FC_NST]);
        }
      }
      for (int d = 0; d < ndst; ++d) {
        uint4* dp = reinterpret_cast<uint4*>(dst[d] + off0 + off);
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int j = lane + 32 * (u + PER * h);
          if (j < nv) dp[j] = v[u];
        }
      }
    }
  }
  rg.seq += (unsigned)npieces;
}

// Reduce `nbytes` (all pointers 16-aligned, multiple of 16): sources are
// bulk-loaded into the ring, 32 lanes sum them and store 16-byte vectors.
template <int DT, bool SC>
__device__ void bulk_reduce(Ring& rg, const char* const* src, int nsrc, char* const* dst,
                            int ndst, long long off0, long long nbytes, int lane, bool scaled,
                            float sc) {
  const long long seg = (long long)(FC_STAGE / nsrc) & ~15LL;  // bytes per source per piece
  const long long npieces = (nbytes + seg - 1) / seg;
  const unsigned base = rg.seq;
  char* const d0 = dst[0] + off0;  // the first destination stays in registers
  if (lane == 0) {
    for (long long i = 0; i < npieces && i < FC_NST - 1; ++i) {
      const unsigned q = base + (unsigned)i;
      const long long off = i * seg;
      const unsigned len = (unsigned)((nbytes - off) < seg ? (nbytes - off) : seg);
      char* sb = rg.buf + (q % FC_NST) * FC_STAGE;
      mbar_expect_tx(&rg.bar[q % FC_NST], len * nsrc);
      for (int s = 0; s < nsrc; ++s)
        bulk_load(sb + s * seg, src[s] + off0 + off, len, &rg.bar[q % FC_NST]);
    }
  }
  for (long long i = 0; i < npieces; ++i) {
    const unsigned q = base + (unsigned)i;
    mbar_wait(&rg.bar[q % FC_NST], (q / FC_NST) & 1u);
    const char* sb = rg.buf + (q % FC_NST) * FC_STAGE;
    const long long off = i * seg;
    const int nv = (int)(((nbytes - off) < seg ? (nbytes - off) : seg) / 16);
    // RU vectors per lane in flight: 4-byte types gain from overlapping
    // independent smem loads (fp32 virtual reduce-scatter 0.976 -> 0.991 of
    // HBM); 2-byte types lose 1 % with two (tools/exp_redu_r02.sh)
    constexpr int RU = sizeof(typename Red<DT>::E) == 2 ? FC_RED_U2 : FC_RED_U;
    for (int j0 = lane; j0 < nv; j0 += 32 * RU) {
      Acc16<DT> acc[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u)
        if (j0 + 32 * u < nv) acc[u].init(reinterpret_cast<const uint4*>(sb)[j0 + 32 * u]);
      for (int s = 1; s < nsrc; ++s) {
        const uint4* ss = reinterpret_cast<const uint4*>(sb + s * seg);
#pragma unroll
        for (int u = 0; u < RU; ++u)
          if (j0 + 32 * u < nv) acc[u].add(ss[j0 + 32 * u]);
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (j0 + 32 * u >= nv) break;
        if constexpr (SC) {
          if (scaled) acc[u].scale(sc);
        }
        const uint4 out = acc[u].pack();
        reinterpret_cast<uint4*>(d0 + off)[j0 + 32 * u] = out;
        for (int d = 1; d < ndst; ++d) reinterpret_cast<uint4*>(dst[d] + off0 + off)[j0 + 32 * u] = out;
      }
    }
    __syncwarp();
    // refill the stage consumed in iteration i-1 (all lanes passed its __syncwarp)
    if (lane == 0 && i + FC_NST - 1 < npieces) {
      const long long p = i + FC_NST - 1;
      const unsigned q2 = base + (unsigned)p;
      const long long off2 = p * seg;
      const unsigned len2 = (unsigned)((nbytes - off2) < seg ? (nbytes - off2) : seg);
      char* sb2 = rg.buf + (q2 % FC_NST) * FC_STAGE;
      fence_proxy_async_smem();  // generic reads of the reused stage before async writes
      mbar_expect_tx(&rg.bar[q2 % FC_NST], len2 * nsrc);
      for (int s = 0; s < nsrc; ++s)
        bulk_load(sb2 + s * seg, src[s] + off0 + off2, len2, &rg.bar[q2 % FC_NST]);
    }
  }
  rg.seq += (unsigned)npieces;
}

struct Geo {
  long long base, lo, hi;
};

// Chunk c of n covers [bound(c), bound(c+1)).  Regular chunks weigh 2^tail;
// the last `tail` chunks halve at each step (2^(tail-1) ... 1), so every
// launch ends on small chunks: the final hops of deep chains and the last
// claims finish sooner.  fc_api.cu (chunk_prefix) sizes scratch windows with
// the same weights.
__device__ __forceinline__ long long chunk_prefix(int c, int n, int tail) {
  const int reg = n - tail;
  const long long w = 1LL << tail;
  if (c <= reg) return w * c;
  return w * reg + (w - (1LL << (tail - (c - reg))));
}

__device__ __forceinline__ long long chunk_bound(const Geo& g, int c, int n, int tail) {
  if (c <= 0) return g.lo;
  if (c >= n) return g.hi;
  const long long len = g.hi - g.lo;
  const long long F = chunk_prefix(n, n, tail);
  long long b = (g.lo + len * chunk_prefix(c, n, tail) / F) & ~(long long)(FC_ALIGN - 1);
  return b < g.lo ? g.lo : b;
}

// SC (AVG kernels only): when `scaled` (a root item), the fp32 sum is
// multiplied by `sc` before the final rounding.  SUM kernels compile it out.
template <int DT, bool SC>
__device__ void move(Ring& rg, const char* const* src, int ns, char* const* dst, int nd,
                     long long nbytes, int esize, int lane, int copy_mode, bool& used_bulk,
                     bool scaled, float sc) {
  if (nbytes <= 0 || nd <= 0) return;
  const uintptr_t a0 = (uintptr_t)src[0];
  uintptr_t diff = 0;
  for (int s = 1; s < ns; ++s) diff |= (uintptr_t)src[s] - a0;
  for (int d = 0; d < nd; ++d) diff |= (uintptr_t)dst[d] - a0;
  if (ns == 1) {
    if ((diff & 15) == 0 && nbytes >= 1024) {
      const long long head = (long long)((16 - (a0 & 15)) & 15);
      const long long body = (nbytes - head) & ~15LL;
      warp_copy(src[0], dst, nd, 0, head, lane);
      if (copy_mode == 0) {
        bulk_copy(rg, src[0], dst, nd, head, body, lane);
        used_bulk = true;
      } else {
        bulk_copy_stg(rg, src[0], dst, nd, head, body, lane);
      }
      warp_copy(src[0], dst, nd, head + body, nbytes - head - body, lane);
    } else {
      warp_copy(src[0], dst, nd, 0, nbytes, lane);
    }
    return;
  }
  if ((diff & 15) == 0) {
    long long head = (long long)((16 - (a0 & 15)) & 15);
    if (head > nbytes) head = nbytes;
    warp_reduce_scalar<DT, SC>(src, ns, dst, nd, 0, head / esize, lane, scaled, sc);
    const long long body = (nbytes - head) & ~15LL;
    if (body > 0) {
      if (ns <= 8 && body >= 1024)
        bulk_reduce<DT, SC>(rg, src, ns, dst, nd, head, body, lane, scaled, sc);
      else
        warp_reduce_vec<DT, SC>(src, ns, dst, nd, head, body / 16, lane, scaled, sc);
    }
    const long long t0 = head + body;
    warp_reduce_scalar<DT, SC>(src, ns, dst, nd, t0, (nbytes - t0) / esize, lane, scaled, sc);
  } else {
    warp_reduce_scalar<DT, SC>(src, ns, dst, nd, 0, nbytes / esize, lane, scaled, sc);
  }
}

// Shared per-CTA item state (one item in flight per CTA).
struct ItemShared {
  int item;
  int ok;
};
// Per-warp source / destination pointer tables of the current item.
struct ItemPtrs {
  const char* src[FC_WPC][FC_MAXS];
  char* dst[FC_WPC][FC_MAXS];
};
// Append `val` to a shared pointer table (lane 0 stores, every lane counts).
#define FC_PUT(arr, cnt, val)        \
  do {                               \
    auto fc_v_ = (val);              \
    if (lane == 0) (arr)[(cnt)] = fc_v_; \
    ++(cnt);                         \
  } while (0)

// One item (task, chunk) executed by the whole CTA: thread 0 waits for the
// inputs, every warp moves a 128-byte-aligned 1/FC_WW sub-range through its
// own bulk ring, and thread 0 publishes after a CTA barrier.
template <int DT, int WW, bool AVG>
__device__ void run_item(const FcParams& P, int me, FcCtl* ctl, const int* T, int c,
                         unsigned e, int w, int lane, unsigned& ready_mask, Ring& rg,
                         ItemShared* sh, ItemPtrs* ptrs, unsigned long long& t_ready,
                         unsigned long long& t_moved, unsigned long long& peer_bytes) {
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
  const long long b0 = chunk_bound(g, c, P.nchunks, P.tail);
  const long long b1 = chunk_bound(g, c + 1, P.nchunks, P.tail);
  const long long wbase = chunk_bound(g, P.c0, P.nchunks, P.tail) & ~(long long)(FC_ALIGN - 1);
  const int fi = c - P.c0;
  unsigned* const myflags = P.flags[me];
  const int n_ag = __ldg(T + TW_N_AG_CHILD);
  const int n_rs = __ldg(T + TW_N_RS_CHILD);
  const int rs_parent = __ldg(T + TW_RS_PARENT);

  // 1. wait for inputs (parent / children flags) and for destination ranks
  //    to have entered this launch (entry barrier, guards buffer reuse).
  const int wl = w % WW;  // warp index within the worker
  const int wk = w / WW;  // worker index within the CTA
  const bool leader = (wl == 0 && lane == 0);
  if (leader) {
    bool ok = true;
    if (kind == FC_K_AG_FWD)
      ok = spin_geq(myflags + P.ag_flag_off + t * P.maxc + fi, e, ctl, P.timeout_ns,
                    FC_DEVERR_TIMEOUT_AG);
    if (kind == FC_K_WAIT_AG) {
      // leaf: every chunk of this launch window has arrived; re-arm the counter
      unsigned* cnt = myflags + P.cnt_off + t;
      ok = spin_geq(cnt, (unsigned)(P.c1 - P.c0), ctl, P.timeout_ns, FC_DEVERR_TIMEOUT_AG);
      if (ok) atomicSub(cnt, (unsigned)(P.c1 - P.c0));
    }
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
          ok = wait_ready(P, me, x, e, ctl);
          if (ok) ready_mask |= 1u << x;
        }
      }
    }
    sh->ok = ok ? 1 : 0;
    if (P.trace) t_ready = globaltimer();
  }
  if (kind == FC_K_WAIT_AG) return;  // uniform: the leader alone waited
  worker_sync<WW>(wk);
  if (!sh->ok) return;

  // 2. move / reduce this warp's share of the chunk
  long long s0 = b0 + (((b1 - b0) * wl / WW) & ~(long long)(FC_ALIGN - 1));
  long long s1 = (wl == WW - 1) ? b1 : b0 + (((b1 - b0) * (wl + 1) / WW) & ~(long long)(FC_ALIGN - 1));
  if (s1 < s0) s1 = s0;
  // this warp's source / destination pointers, in shared memory: filled by
  // lane 0, read by every lane (no local-memory arrays, no spills)
  const char** const src = ptrs->src[w];
  char** const dst = ptrs->dst[w];
  int ns = 0, nd = 0;
  const long long slot_phase = s0 - wbase;
  __syncwarp();  // the previous item's readers are done with the table
  if (kind == FC_K_AG_ROOT || kind == FC_K_AG_FWD) {
    const char* first = (kind == FC_K_AG_ROOT) ? P.send[me] + (s0 - g.base) : P.recv[me] + s0;
    FC_PUT(src, ns, first);
    if (kind == FC_K_AG_ROOT && !P.root_local_done && P.recv[me] + s0 != first)
      FC_PUT(dst, nd, P.recv[me] + s0);
    for (int j = 0; j < n_ag; ++j) FC_PUT(dst, nd, P.recv[__ldg(T + TW_AG_CHILD + j)] + s0);
  } else {
    FC_PUT(src, ns, P.send[me] + s0);
    for (int j = 0; j < n_rs; ++j)
      FC_PUT(src, ns, P.scratch[me] + P.unit_bytes * __ldg(T + TW_RS_CPREFIX + j) +
                  2LL * FC_ALIGN * __ldg(T + TW_RS_CSLOT + j) + slot_phase);
    if (kind == FC_K_RS_FWD) {
      FC_PUT(dst, nd, P.scratch[rs_parent] + P.unit_bytes * __ldg(T + TW_RS_PPREFIX) +
                  2LL * FC_ALIGN * __ldg(T + TW_RS_PSLOT) + slot_phase);
    } else if (kind == FC_K_RS_ROOT) {
      FC_PUT(dst, nd, P.recv[me] + (s0 - g.base));
    } else {  // FC_K_AR_ROOT
      FC_PUT(dst, nd, P.recv[me] + s0);
      for (int j = 0; j < n_ag; ++j) FC_PUT(dst, nd, P.recv[__ldg(T + TW_AG_CHILD + j)] + s0);
    }
  }
  __syncwarp();  // table complete before any lane reads it
  bool used_bulk = false;
  // AVG: the root scales its fp32 sum once, before the final rounding
  move<DT, AVG>(rg, src, ns, dst, nd, s1 - s0, P.esize, lane, P.copy_mode, used_bulk,
                AVG && (kind == FC_K_RS_ROOT || kind == FC_K_AR_ROOT), P.scale);
  if (used_bulk && lane == 0) {
    bulk_wait_all();
    fence_proxy_async_global();
  }

  // 3. publish: the CTA barrier orders every thread's stores (and the bulk
  //    completions above) before thread 0's cumulative .sys release.
  worker_sync<WW>(wk);
  if (P.trace && leader) {
    t_moved = globaltimer();
    // bytes this item stored into other ranks: the chunk to every remote
    // destination, plus one 4-byte flag per child / parent
    int remote = 0;
    if (kind == FC_K_RS_FWD) remote = (rs_parent != me);
    else if (kind != FC_K_RS_ROOT)
      for (int j = 0; j < n_ag; ++j) remote += (__ldg(T + TW_AG_CHILD + j) != me);
    peer_bytes = (unsigned long long)(b1 - b0) * remote + 4ull * remote;
  }
  if (kind == FC_K_RS_ROOT || !leader) return;
  if (kind == FC_K_RS_FWD) {
    st_release_sys(P.flags[rs_parent] + P.rs_flag_off + __ldg(T + TW_RS_PSLOT) * P.maxc + fi, e);
  } else {
    const int leaves = __ldg(T + TW_AG_LEAFMASK);
    for (int j = 0; j < n_ag; ++j) {
      unsigned* f = P.flags[__ldg(T + TW_AG_CHILD + j)];
      if ((leaves >> j) & 1)
        red_release_sys_add(f + P.cnt_off + t, 1u);
      else
        st_release_sys(f + P.ag_flag_off + t * P.maxc + fi, e);
    }
  }
}

#define FC_LL_UNROLL 8  // 4-line batches per warp iteration (32 lines = 3.75 KiB payload)

// Poll FC_LL_UNROLL 4-line batches (lane group g = lane/8 owns line base+4u+g)
// until every valid line carries `flag`.  Returns false on timeout / error.
__device__ __forceinline__ bool ll_poll(const char* const* line, const bool* valid,
                                        unsigned long long flag, int lane,
                                        unsigned long long* a, unsigned long long* b,
                                        FcCtl* ctl, long long timeout_ns) {
  unsigned long long t0 = 0;
  for (unsigned it = 0;; ++it) {
#pragma unroll
    for (int u = 0; u < FC_LL_UNROLL; ++u)
      if (valid[u]) ld_line16(line[u], a[u], b[u]);
    int mine = 1;
#pragma unroll
    for (int u = 0; u < FC_LL_UNROLL; ++u)
      mine &= (!valid[u] || (lane & 7) != 7 || b[u] == flag) ? 1 : 0;
    const int grp = __shfl_sync(0xffffffffu, mine, (lane & ~7) | 7);
    if (__all_sync(0xffffffffu, grp)) return true;
    if ((it & 255u) == 255u) {
      int bad = 0;
      if (lane == 0) {
        if (!t0) t0 = globaltimer();
        if (ld_volatile(&ctl->error) != 0) bad = 1;
        else if ((long long)(globaltimer() - t0) > timeout_ns) {
          atomicCAS(&ctl->error, 0u, (unsigned)FC_DEVERR_TIMEOUT_AG);
          bad = 1;
        }
      }
      if (__shfl_sync(0xffffffffu, bad, 0)) return false;
    }
  }
}

// One item in the LL protocol.  Lines of the chunk are dealt to the worker's
// warps 4*FC_LL_UNROLL at a time; lane group g (8 lanes) handles one 128-byte
// line per batch, with all batches' loads in flight together.
template <int DT, int WW, bool AVG>
__device__ void run_item_ll(const FcParams& P, int me, FcCtl* ctl, const int* T, int c,
                            unsigned e, int w, int lane, unsigned& ready_mask, ItemShared* sh,
                            ItemPtrs* ptrs, unsigned long long& t_ready,
                            unsigned long long& peer_bytes) {
  constexpr int U = FC_LL_UNROLL;
  const int kind = __ldg(T + TW_KIND);
  const int root = __ldg(T + TW_ROOT);
  const long long es = P.esize;
  long long Sr = P.total_elems - (long long)root * P.stride_elems;
  Sr = Sr < 0 ? 0 : (Sr > P.shard_elems ? P.shard_elems : Sr);
  const long long base = (long long)root * P.stride_elems * es;
  const long long lo = base + (Sr * __ldg(T + TW_MLO) / P.k) * es;
  const long long hi = base + (Sr * __ldg(T + TW_MHI) / P.k) * es;
  const long long L = (hi - lo + FC_LL_PAY - 1) / FC_LL_PAY;
  const long long l0 = L * c / P.nchunks, l1 = L * (c + 1) / P.nchunks;
  const long long lw = L * P.c0 / P.nchunks;
  const int n_ag = __ldg(T + TW_N_AG_CHILD);
  const int n_rs = __ldg(T + TW_N_RS_CHILD);
  const int rs_parent = __ldg(T + TW_RS_PARENT);
  const int wl = w % WW;
  const int wk = w / WW;
  const bool leader = (wl == 0 && lane == 0);
  const unsigned long long flag = (unsigned long long)e;

  // No entry wait.  LL stores only ever land in peers' staging, never in user
  // buffers, and staging alternates between two halves by epoch parity.  A
  // rank in launch e has finished e-1, which needed every rank's data (every
  // rank roots a non-empty tree, or feeds one that reaches every rank), so
  // every rank has finished e-2, the last user of this half.  Lines left there
  // carry epoch e-2, never e.
  (void)ready_mask;
  if (P.trace && leader) t_ready = globaltimer();

  const int g = lane >> 3, gl = lane & 7;
  const long long slot_ofs = -lw * 128LL;  // line l of the window at slot + (l - lw)*128
  const long long ll_off = P.ll_region_off + (long long)(e & 1u) * P.ll_half;
  auto slot_ptr = [&](int rank, long long region, int slot, int prefix) -> char* {
    return P.scratch[rank] + ll_off + region + P.ll_unit_bytes * prefix + 256LL * slot + slot_ofs;
  };
  const bool polls = (kind == FC_K_AG_FWD || kind == FC_K_WAIT_AG);
  const char* my_ag = polls ? slot_ptr(me, P.ll_ag_base, __ldg(T + TW_AG_MYSLOT),
                                       __ldg(T + TW_AG_MYPREFIX)) : nullptr;
  // payload words of this lane in a line: gl<7 -> 2*gl, 2*gl+1 ; gl==7 -> 14 (+flag)
  const int q0 = 2 * gl;
  const bool two = gl != 7;
  const char* local_src = nullptr;  // payload source, indexed by absolute byte offset
  if (kind == FC_K_AG_ROOT) local_src = P.send[me] - base;
  if (kind == FC_K_RS_FWD || kind == FC_K_RS_ROOT || kind == FC_K_AR_ROOT) local_src = P.send[me];
  char* out_local = nullptr;  // payload destination in a local buffer
  if (polls || kind == FC_K_AR_ROOT) out_local = P.recv[me];
  if (kind == FC_K_AG_ROOT && !P.root_local_done && P.recv[me] + lo != P.send[me] + (lo - base))
    out_local = P.recv[me];
  if (kind == FC_K_RS_ROOT) out_local = P.recv[me] - base;  // out has S elements
  // payload offsets (pay + 8*q0) are lo plus multiples of 8: the local
  // buffers' alignment at lo (8, 4 or any) picks the access width
  // (warp-uniform)
  auto acls = [&](const char* b) -> int {
    if (!b) return 8;
    const uintptr_t a = (uintptr_t)(b + lo);
    return (a & 7) == 0 ? 8 : ((a & 3) == 0 ? 4 : 1);
  };
  const int align = min(acls(local_src), acls(out_local));

  // the line loop, instantiated per alignment class: 8 (one 8-byte access),
  // 4 (two 4-byte accesses; odd fp32 counts, offset views) -- both without
  // branches, so all loads of a batch are in flight together -- and any
  auto lines = [&](auto aligned) -> bool {
    constexpr int AL = decltype(aligned)::value;
    for (long long lb = l0 + 4LL * U * wl; lb < l1; lb += 4LL * U * WW) {
      bool valid[U], v0[U], v1[U];
      long long pay[U];
      unsigned long long w0[U], w1[U];
      // a slice whose length is not a multiple of 8 ends in a partial word:
      // n0/n1 its bytes (zero-padded in the line), only the last line has one
      int n0 = 0, n1 = 0;
  #pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long l = lb + 4 * u + g;
        valid[u] = l < l1;
        pay[u] = lo + (long long)FC_LL_PAY * l;
        v0[u] = valid[u] && pay[u] + 8LL * q0 + 8 <= hi;
        v1[u] = valid[u] && two && pay[u] + 8LL * (q0 + 1) + 8 <= hi;
        if (valid[u] && !v0[u] && pay[u] + 8LL * q0 < hi) n0 = (int)(hi - pay[u] - 8LL * q0);
        if (valid[u] && two && !v1[u] && pay[u] + 8LL * (q0 + 1) < hi)
          n1 = (int)(hi - pay[u] - 8LL * (q0 + 1));
        w0[u] = 0;
        w1[u] = 0;
      }
      // the line holding the slice's last byte (its partial word, if any)
      const long long tl = (hi - lo - 1) / FC_LL_PAY;
      if (polls) {
        const char* lp[U];
  #pragma unroll
        for (int u = 0; u < U; ++u) lp[u] = my_ag + (lb + 4 * u + g) * 128 + 16 * gl;
        if (!ll_poll(lp, valid, flag, lane, w0, w1, ctl, P.timeout_ns)) return false;
      } else {
  #pragma unroll
        for (int u = 0; u < U; ++u) {
          const char* src = local_src + pay[u] + 8 * q0;  // rank-local buffer, any alignment
          if constexpr (AL == 8) {  // aligned bases: every line's loads in flight together
            if (v0[u]) w0[u] = __ldcg(reinterpret_cast<const unsigned long long*>(src));
            if (v1[u]) w1[u] = __ldcg(reinterpret_cast<const unsigned long long*>(src) + 1);
          } else if constexpr (AL == 4) {
            const unsigned* q = reinterpret_cast<const unsigned*>(src);
            if (v0[u]) w0[u] = (unsigned long long)__ldcg(q) | ((unsigned long long)__ldcg(q + 1) << 32);
            if (v1[u]) w1[u] = (unsigned long long)__ldcg(q + 2) | ((unsigned long long)__ldcg(q + 3) << 32);
          } else {
            if (v0[u]) w0[u] = ld_u64_any(src);
            if (v1[u]) w1[u] = ld_u64_any(src + 8);
          }
          if (lb + 4 * u + g == tl) {
            if (n0) w0[u] = ld_tail(src, n0);
            if (n1) w1[u] = ld_tail(src + 8, n1);
          }
        }
        if (kind != FC_K_AG_ROOT && n_rs > 0) {
          Acc8<DT> a0[U], a1[U];
  #pragma unroll
          for (int u = 0; u < U; ++u) {
            a0[u].init(w0[u]);
            a1[u].init(w1[u]);
          }
          for (int j = 0; j < n_rs; ++j) {
            const char* cl = slot_ptr(me, 0, __ldg(T + TW_RS_CSLOT + j), __ldg(T + TW_RS_CPREFIX + j));
            const char* lp[U];
            unsigned long long x0[U], x1[U];
  #pragma unroll
            for (int u = 0; u < U; ++u) lp[u] = cl + (lb + 4 * u + g) * 128 + 16 * gl;
            if (!ll_poll(lp, valid, flag, lane, x0, x1, ctl, P.timeout_ns)) return false;
  #pragma unroll
            for (int u = 0; u < U; ++u) {
              a0[u].add(x0[u]);
              a1[u].add(x1[u]);
            }
          }
          if (AVG && kind != FC_K_RS_FWD) {  // root: scale the fp32 sum once
  #pragma unroll
            for (int u = 0; u < U; ++u) {
              a0[u].scale(P.scale);
              a1[u].scale(P.scale);
            }
          }
  #pragma unroll
          for (int u = 0; u < U; ++u) {
            w0[u] = a0[u].pack();
            w1[u] = a1[u].pack();
          }
        }
      }
      // local payload write
      if (out_local) {
  #pragma unroll
        for (int u = 0; u < U; ++u) {
          char* o = out_local + pay[u] + 8 * q0;
          if constexpr (AL == 8) {
            if (v0[u]) reinterpret_cast<unsigned long long*>(o)[0] = w0[u];
            if (v1[u]) reinterpret_cast<unsigned long long*>(o)[1] = w1[u];
          } else if constexpr (AL == 4) {
            unsigned* q = reinterpret_cast<unsigned*>(o);
            if (v0[u]) {
              q[0] = (unsigned)w0[u];
              q[1] = (unsigned)(w0[u] >> 32);
            }
            if (v1[u]) {
              q[2] = (unsigned)w1[u];
              q[3] = (unsigned)(w1[u] >> 32);
            }
          } else {
            if (v0[u]) st_u64_any(o, w0[u]);
            if (v1[u]) st_u64_any(o + 8, w1[u]);
          }
          if (lb + 4 * u + g == tl) {
            if (n0) st_tail(o, w0[u], n0);
            if (n1) st_tail(o + 8, w1[u], n1);
          }
        }
      }
      // line stores to peers' staging (a per-batch local table measures 13 %
      // faster at 64 MiB than a shared-memory one built once per item)
      char* dl[FC_MAXS];
      int nl = 0;
      if (kind == FC_K_RS_FWD) {
        dl[nl++] = slot_ptr(rs_parent, 0, __ldg(T + TW_RS_PSLOT), __ldg(T + TW_RS_PPREFIX));
      } else if (kind == FC_K_AG_ROOT || kind == FC_K_AG_FWD || kind == FC_K_AR_ROOT) {
        for (int j = 0; j < n_ag; ++j)
          dl[nl++] = slot_ptr(__ldg(T + TW_AG_CHILD + j), P.ll_ag_base, __ldg(T + TW_AG_CSLOT + j),
                              __ldg(T + TW_AG_CPREFIX + j));
      }
      // one warp-wide store per line: the partial-word loads above diverge,
      // and a line whose 8 lane stores issued apart could show its flag
      // before its payload
      __syncwarp();
      for (int d = 0; d < nl; ++d) {
  #pragma unroll
        for (int u = 0; u < U; ++u)
          if (valid[u])
            st_line16(dl[d] + (lb + 4 * u + g) * 128 + 16 * gl, w0[u], two ? w1[u] : flag);
      }
    }
    return true;
  };
  const bool ok = align == 8   ? lines(std::integral_constant<int, 8>{})
                  : align == 4 ? lines(std::integral_constant<int, 4>{})
                               : lines(std::integral_constant<int, 1>{});
  if (!ok) return;
  if (P.trace && leader) {  // 128-byte lines of this chunk to every peer destination
    int remote = 0;
    if (kind == FC_K_RS_FWD) remote = (rs_parent != me);
    else if (kind == FC_K_AG_ROOT || kind == FC_K_AG_FWD || kind == FC_K_AR_ROOT)
      for (int j = 0; j < n_ag; ++j) remote += (__ldg(T + TW_AG_CHILD + j) != me);
    peer_bytes = (unsigned long long)(l1 - l0) * 128ull * remote;
  }
  worker_sync<WW>(wk);
}

template <int DT, int WW, int PROTO, bool AVG>
__global__ void __launch_bounds__(FC_BLOCK, 1) fc_forest_kernel(const __grid_constant__ FcParams P) {
  constexpr int FC_NWK = FC_WPC / WW;
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bars[FC_WPC * FC_NST];
  __shared__ unsigned s_epoch;
  __shared__ ItemShared sh_all[FC_NWK];
  __shared__ ItemPtrs s_ptrs;
  const int lr = blockIdx.x / P.ctas_per_rank;
  const int me = P.local_rank[lr];
  FcCtl* const ctl = P.ctl[lr];
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < FC_WPC * FC_NST) mbar_init(&bars[threadIdx.x], 1);
  // programmatic dependent launch: the prologue above overlaps the previous
  // kernel's tail; everything below waits for it to complete (no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) s_epoch = ld_volatile(&ctl->epoch) + 1;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const unsigned e = s_epoch;
  // entry barrier: tell every peer that this rank entered launch e, and with
  // which output buffer (the tag store is ordered before the release)
  if ((int)threadIdx.x < P.nranks && (int)threadIdx.x != me) {
    unsigned long long* pf = reinterpret_cast<unsigned long long*>(P.flags[threadIdx.x]);
    st_release_sys64(pf + me, ((unsigned long long)tag32(P) << 32) | e);
  }

  const int wk = w / WW;
  const bool lead = (w % WW == 0) && lane == 0;
  ItemShared& sh = sh_all[wk];
  Ring rg;
  rg.buf = smem + (size_t)w * FC_NST * FC_STAGE;
  rg.bar = &bars[w * FC_NST];
  rg.seq = 0;
  const int* const tasks = P.tasks[lr];
  const int nact = P.nactive[lr];
  const int nwait = P.nwait[lr];
  const long long W = P.c1 - P.c0;
  const long long span = W + (long long)P.lag * P.lag_max[lr];
  // LL: leaf tasks are real items (they copy their lines out of staging)
  const int nitem = PROTO ? nact + nwait : nact;
  const long long nA = (long long)nitem * span;
  const long long total = nA + (PROTO ? 0 : nwait);  // simple: one completion wait per leaf
  unsigned ready_mask = 1u << me;
  FcTraceRec* const trace = P.trace;
  // Claim one item at a time.  (Claiming one ahead hides the atomic's round
  // trip but strands a claimed item behind a busy worker: measured -20 % at
  // 4-64 MiB on 4 GPUs and -2 % at N=1, for -0.5 us on tiny calls.)
  for (;;) {
    if (lead) {
      int v = (int)atomicAdd(&ctl->claim, 1u);
      if (ld_volatile(&ctl->error) != 0) v = INT_MAX;
      sh.item = v;
    }
    worker_sync<WW>(wk);
    const long long item = sh.item;
    worker_sync<WW>(wk);  // sh.item is rewritten by the next claim
    if (item >= total) break;
    int c, ti;
    if (item < nA) {
      const long long d = item / nitem;
      ti = (int)(item - d * nitem);
      const long long cc =
          d - (long long)P.lag * __ldg(tasks + (long long)ti * FC_TASK_WORDS + TW_LAG);
      if (cc < 0 || cc >= W) continue;  // outside this task's diagonal window
      c = (int)cc;
    } else {
      c = (int)(W - 1);
      ti = nact + (int)(item - nA);
    }
    const unsigned long long t0 = trace ? globaltimer() : 0;
    unsigned long long t_ready = t0, t_moved = t0, peer_bytes = 0;
    if constexpr (PROTO == 1)
      run_item_ll<DT, WW, AVG>(P, me, ctl, tasks + (long long)ti * FC_TASK_WORDS, P.c0 + c, e, w,
                          lane, ready_mask, &sh, &s_ptrs, t_ready, peer_bytes);
    else
      run_item<DT, WW, AVG>(P, me, ctl, tasks + (long long)ti * FC_TASK_WORDS, P.c0 + c, e, w, lane,
                       ready_mask, rg, &sh, &s_ptrs, t_ready, t_moved, peer_bytes);
    if (trace && lead) {
      const unsigned idx = atomicAdd(P.trace_count, 1u);
      if (idx < P.trace_cap) {
        FcTraceRec r;
        r.t_start = t0;
        r.t_end = globaltimer();
        r.t_wait = (unsigned)(t_ready - t0);
        r.t_move = t_moved > t_ready ? (unsigned)(t_moved - t_ready) : 0u;
        r.peer_bytes = peer_bytes > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned)peer_bytes;
        r.chunk = P.c0 + c;
        r.rank = (short)me;
        r.task = (short)ti;
        r.worker = (short)((blockIdx.x % P.ctas_per_rank) * FC_NWK + wk);
        r.launch = (unsigned short)e;
        trace[idx] = r;
      }
    }
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // The last CTA of this rank re-arms the counters and publishes the epoch.
  // No fences: every CTA's claims returned before its `done` increment, and
  // the next launch reads these words only after this grid has completed.
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&ctl->done, 1u);
    if (prev == (unsigned)P.ctas_per_rank - 1u) {
      ctl->claim = 0;
      ctl->done = 0;
      atomicExch(&ctl->epoch, e);
    }
  }
}


}  // namespace

// Kernel pointer for one (dtype, worker warps, protocol, AVG) instantiation.
#define FC_DEFINE_KERNEL_TABLE(NAME, DT, AVG)                                     \
  const void* NAME(int ww, int proto) {                                           \
    if (proto) {                                                                  \
      switch (ww) {                                                               \
        case 1: return (const void*)fc_forest_kernel<DT, 1, 1, AVG>;              \
        case 2: return (const void*)fc_forest_kernel<DT, 2, 1, AVG>;              \
        case 4: return (const void*)fc_forest_kernel<DT, 4, 1, AVG>;              \
        default: return (const void*)fc_forest_kernel<DT, 8, 1, AVG>;             \
      }                                                                           \
    }                                                                             \
    switch (ww) {                                                                 \
      case 1: return (const void*)fc_forest_kernel<DT, 1, 0, AVG>;                \
      case 2: return (const void*)fc_forest_kernel<DT, 2, 0, AVG>;                \
      case 4: return (const void*)fc_forest_kernel<DT, 4, 0, AVG>;                \
      default: return (const void*)fc_forest_kernel<DT, 8, 0, AVG>;               \
    }                                                                             \
  }
