// Microbenchmark: per-SM copy bandwidth local->peer over NVLink (and local->
// local) for the data-movement primitives the forest kernel can use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_p2p tools/mb_p2p.cu
//   ./mb_p2p [bytes_per_cta_MiB]
// Modes: 0 LDG/STG (256 thr, unroll 8), 1 TMA load -> smem -> STG,
//        2 TMA load -> smem -> TMA store, 3 LDG/STG 1024 thr unroll 4
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_ldst(const uint4* __restrict__ src, uint4* dst, long long nvec_per_cta) {
  const uint4* s = src + blockIdx.x * nvec_per_cta;
  uint4* d = dst + blockIdx.x * nvec_per_cta;
  constexpr int U = 8;
  for (long long i = threadIdx.x; i < nvec_per_cta; i += (long long)blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = i + (long long)u * blockDim.x; if (j < nvec_per_cta) v[u] = __ldcg(s + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = i + (long long)u * blockDim.x; if (j < nvec_per_cta) d[j] = v[u]; }
  }
}

template <int NST, int STAGE, bool TMA_STORE>
__global__ void k_tma(const char* __restrict__ src, char* dst, long long bytes_per_cta) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[32][NST];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) for (int s = 0; s < NST; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[w][s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  char* ring = smem + (size_t)w * NST * STAGE;
  // each warp owns a contiguous slice
  const long long per_w = (bytes_per_cta / nw) / STAGE * STAGE;
  const char* s = src + blockIdx.x * bytes_per_cta + w * per_w;
  char* d = dst + blockIdx.x * bytes_per_cta + w * per_w;
  const long long np = per_w / STAGE;
  auto issue = [&](long long p) {
    const int st = p % NST;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[w][st])), "r"(STAGE));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(ring + st * STAGE)), "l"(s + p * STAGE), "r"(STAGE), "r"(smem_u32(&bar[w][st])) : "memory");
  };
  if (lane == 0) for (long long p = 0; p < np && p < NST - 1; ++p) issue(p);
  for (long long p = 0; p < np; ++p) {
    const int st = p % NST;
    const unsigned par = (p / NST) & 1;
    unsigned ok = 0;
    while (!ok) asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }" : "=r"(ok) : "r"(smem_u32(&bar[w][st])), "r"(par) : "memory");
    if (TMA_STORE) {
      if (lane == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(d + p * STAGE), "r"(smem_u32(ring + st * STAGE)), "r"(STAGE) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (p + NST - 1 < np) { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); issue(p + NST - 1); }
      }
    } else {
      const uint4* sb = reinterpret_cast<const uint4*>(ring + st * STAGE);
      constexpr int PER = STAGE / 16 / 32;
      uint4 v[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) v[u] = sb[lane + 32 * u];
      __syncwarp();
      if (lane == 0 && p + NST - 1 < np) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(p + NST - 1); }
      uint4* dp = reinterpret_cast<uint4*>(d + p * STAGE);
#pragma unroll
      for (int u = 0; u < PER; ++u) dp[lane + 32 * u] = v[u];
    }
  }
  if (TMA_STORE && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const long long per_cta = (argc > 1 ? atoll(argv[1]) : 8) << 20;
  int ndev; CK(cudaGetDeviceCount(&ndev));
  CK(cudaSetDevice(0));
  int can = 0;
  if (ndev > 1) { CK(cudaDeviceCanAccessPeer(&can, 0, 1)); if (can) CK(cudaDeviceEnablePeerAccess(1, 0)); }
  const int maxc = 148;
  const size_t bytes = per_cta * maxc;
  char *src, *dloc, *dpeer = nullptr;
  CK(cudaMalloc(&src, bytes)); CK(cudaMalloc(&dloc, bytes));
  CK(cudaMemset(src, 1, bytes));
  if (can) { CK(cudaSetDevice(1)); CK(cudaMalloc(&dpeer, bytes)); CK(cudaSetDevice(0)); }
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  auto smemset = [](const void* f, int s) { CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, s)); };
  smemset((const void*)k_tma<3, 8192, false>, 8 * 3 * 8192);
  smemset((const void*)k_tma<3, 8192, true>, 8 * 3 * 8192);
  smemset((const void*)k_tma<4, 16384, false>, 3 * 4 * 16384);
  smemset((const void*)k_tma<4, 16384, true>, 3 * 4 * 16384);
  smemset((const void*)k_tma<6, 32768, true>, 1 * 6 * 32768);
  const char* names[] = {"ldst256u8", "ldst512u8", "tma8x3x8K+stg", "tma8x3x8K+tmast", "tma3x4x16K+stg", "tma3x4x16K+tmast", "tma1x6x32K+tmast"};
  for (int target = 0; target < 2; ++target) {
    char* dst = target ? dpeer : dloc;
    if (!dst) continue;
    printf("== %s\n", target ? "peer (NVLink)" : "local");
    for (int mode = 0; mode < 7; ++mode) {
      printf("%-18s", names[mode]);
      for (int ctas : {1, 2, 4, 8, 16, 32, 64, 148}) {
        auto launch = [&]() {
          switch (mode) {
            case 0: k_ldst<<<ctas, 256>>>((const uint4*)src, (uint4*)dst, per_cta / 16); break;
            case 1: k_ldst<<<ctas, 512>>>((const uint4*)src, (uint4*)dst, per_cta / 16); break;
            case 2: k_tma<3, 8192, false><<<ctas, 256, 8 * 3 * 8192>>>(src, dst, per_cta); break;
            case 3: k_tma<3, 8192, true><<<ctas, 256, 8 * 3 * 8192>>>(src, dst, per_cta); break;
            case 4: k_tma<4, 16384, false><<<ctas, 96, 3 * 4 * 16384>>>(src, dst, per_cta); break;
            case 5: k_tma<4, 16384, true><<<ctas, 96, 3 * 4 * 16384>>>(src, dst, per_cta); break;
            case 6: k_tma<6, 32768, true><<<ctas, 32, 6 * 32768>>>(src, dst, per_cta); break;
          }
        };
        launch(); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        for (int it = 0; it < 5; ++it) launch();
        CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        const double gbs = (double)per_cta * ctas * 5 / (ms * 1e-3) / 1e9;
        printf(" %4d:%7.1f", ctas, gbs);
      }
      printf("\n");
    }
  }
  return 0;
}
