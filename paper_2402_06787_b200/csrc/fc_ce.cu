// Copy-engine executor for the 2-rank forest (nvswitch(2): each root's tree
// is the single edge root -> peer).
//
// Moving a shard across that edge is one contiguous copy into the peer's
// registered output, which the GPU's copy engines perform at 745 GB/s per
// direction with both GPUs sending (tools/mb_ce.cu), against 681-714 GB/s
// for SM stores.  The SMs then only synchronise and place the own shard:
//
//   side stream:  fc_ce_copy_kernel      own shard -> own output slot (HBM)
//   stream:       fc_ce_sync_kernel(0)   entry: publish (tag | epoch) to the
//                                        peer, wait for the peer's, check tags
//                 cudaMemcpyAsync        own shard -> peer's output (NVLink CE)
//                 fc_ce_sync_kernel(1)   exit: system fence, publish "done",
//                                        wait for the peer's, bump the epoch
//
// Epochs come from device memory (the control block every engine shares), so
// the sequence captures into a CUDA graph and replays correctly.  Only the
// 2-rank single-switch forest takes this path (fc_api.cu run()).
#include <cuda_runtime.h>

#include <cstdint>

#include "fc_internal.h"

namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until the 64-bit slot's low word reaches e; returns the slot value, or
// 0 with the sticky error set on timeout.
__device__ unsigned long long wait_slot(const unsigned long long* f, unsigned e, FcCtl* ctl,
                                        long long timeout_ns, unsigned code) {
  unsigned long long v = ld_acquire_sys64(f);
  if ((int)((unsigned)v - e) >= 0) return v;
  const unsigned long long t0 = globaltimer();
  for (unsigned i = 1;; ++i) {
    v = ld_acquire_sys64(f);
    if ((int)((unsigned)v - e) >= 0) return v;
    if ((i & 1023u) == 0 && (long long)(globaltimer() - t0) > timeout_ns) {
      if (atomicCAS(&ctl->error, 0u, code) == 0u) {
        ctl->info[0] = (unsigned)(uintptr_t)f;
        ctl->info[1] = e;
        ctl->info[2] = (unsigned)v;
      }
      return 0;
    }
  }
}

__global__ void fc_ce_sync_kernel(const __grid_constant__ FcCeParams P) {
  if (threadIdx.x != 0) return;
  FcCtl* ctl = P.ctl;
  const unsigned e = *reinterpret_cast<volatile unsigned*>(&ctl->epoch) + 1;
  const unsigned tag = (unsigned)(P.tag ^ (P.tag >> 32));
  if (P.phase == 0) {
    // entry: the peer may store into our output once we entered launch e,
    // and we into its output once it did; both must name the same buffer
    st_release_sys64(P.peer_slots + FC_CE_READY + P.me, ((unsigned long long)tag << 32) | e);
    const unsigned long long v =
        wait_slot(P.my_slots + FC_CE_READY + P.peer, e, ctl, P.timeout_ns, FC_DEVERR_TIMEOUT_READY);
    if (v && (unsigned)v == e && (unsigned)(v >> 32) != tag &&
        atomicCAS(&ctl->error, 0u, (unsigned)FC_DEVERR_BUFFER_MISMATCH) == 0u) {
      ctl->info[0] = (unsigned)P.peer;
      ctl->info[1] = tag;
      ctl->info[2] = (unsigned)(v >> 32);
    }
  } else {
    // exit: the copy engine's stores to the peer precede this kernel in
    // stream order; the system-scope fence orders them before the release
    asm volatile("fence.sc.sys;" ::: "memory");
    st_release_sys64(P.peer_slots + FC_CE_DONE + P.me, (unsigned long long)e);
    wait_slot(P.my_slots + FC_CE_DONE + P.peer, e, ctl, P.timeout_ns, FC_DEVERR_TIMEOUT_AG);
    atomicExch(&ctl->epoch, e);
  }
}

// dst <- src (the own shard into the own output slot), 16-byte vectors when
// both are 16-byte aligned, bytes otherwise.
__global__ void __launch_bounds__(512) fc_ce_copy_kernel(char* dst, const char* src, long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const long long nv = n / 16;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (long long i = tid; i < nv; i += 4 * nth) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * nth < nv) v[u] = __ldcs(s + i + u * nth);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * nth < nv) __stcs(d + i + u * nth, v[u]);
    }
    for (long long i = nv * 16 + tid; i < n; i += nth) dst[i] = src[i];
  } else {
    for (long long i = tid; i < n; i += nth) dst[i] = src[i];
  }
}

}  // namespace

int fc_ce_sync_launch(const FcCeParams& p, void* stream) {
  void* args[] = {(void*)&p};
  return (int)cudaLaunchKernel((const void*)fc_ce_sync_kernel, dim3(1), dim3(32), args, 0,
                               (cudaStream_t)stream);
}

int fc_ce_copy_launch(void* dst, const void* src, long long n, int ctas, void* stream) {
  if (n <= 0 || dst == src) return 0;
  fc_ce_copy_kernel<<<ctas, 512, 0, (cudaStream_t)stream>>>((char*)dst, (const char*)src, n);
  return (int)cudaGetLastError();
}
