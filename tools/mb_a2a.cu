// Microbenchmark: per-GPU NVLink egress when every GPU writes to every other
// GPU at once (the traffic pattern of a collective over NVSwitch).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_a2a tools/mb_a2a.cu
//   ./mb_a2a [MiB per peer]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

struct Dsts { uint4* d[8]; };

// grid = npeers * ctas_per_peer; CTA group p writes src -> dst[p]
__global__ void k_push(const uint4* __restrict__ src, Dsts dsts, int ctas_per_peer, long long nvec) {
  const int p = blockIdx.x / ctas_per_peer, b = blockIdx.x % ctas_per_peer;
  uint4* d = dsts.d[p];
  const long long per = nvec / ctas_per_peer;
  const uint4* s = src + b * per;
  d += b * per;
  constexpr int U = 8;
  for (long long i = threadIdx.x; i < per; i += (long long)blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = i + (long long)u * blockDim.x; if (j < per) v[u] = __ldcg(s + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = i + (long long)u * blockDim.x; if (j < per) d[j] = v[u]; }
  }
}

// pull: CTA group p reads peer p's buffer and writes locally
struct Srcs { const uint4* s[8]; };
__global__ void k_pull(Srcs srcs, uint4* dst, int ctas_per_peer, long long nvec) {
  const int p = blockIdx.x / ctas_per_peer, b = blockIdx.x % ctas_per_peer;
  const long long per = nvec / ctas_per_peer;
  const uint4* s = srcs.s[p] + b * per;
  uint4* d = dst + (long long)p * nvec + b * per;
  constexpr int U = 8;
  for (long long i = threadIdx.x; i < per; i += (long long)blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = i + (long long)u * blockDim.x; if (j < per) v[u] = __ldcg(s + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = i + (long long)u * blockDim.x; if (j < per) d[j] = v[u]; }
  }
}

int main(int argc, char** argv) {
  const long long bytes = (argc > 1 ? atoll(argv[1]) : 256) << 20;
  int n; CK(cudaGetDeviceCount(&n));
  if (n > 8) n = 8;
  std::vector<char*> src(n), dst(n);  // dst[d] holds n slots of `bytes`
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < n; ++p) if (p != d) { int ok; CK(cudaDeviceCanAccessPeer(&ok, d, p)); if (ok) cudaDeviceEnablePeerAccess(p, 0); }
    CK(cudaMalloc(&src[d], bytes));
    CK(cudaMalloc(&dst[d], bytes * n));
    CK(cudaMemset(src[d], 1, bytes));
  }
  std::vector<cudaStream_t> st(n);
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaStreamCreate(&st[d])); CK(cudaEventCreate(&e0[d])); CK(cudaEventCreate(&e1[d])); }
  for (int npeers = 1; npeers < n; ++npeers) {
    for (int cpp : {4, 8, 16, 32, 48}) {
      if (cpp * npeers > 148) continue;
      auto run = [&]() {
        for (int d = 0; d < n; ++d) {
          CK(cudaSetDevice(d));
          Dsts ds;
          for (int j = 0; j < npeers; ++j) { int p = (d + 1 + j) % n; ds.d[j] = (uint4*)(dst[p] + (size_t)d * bytes); }
          k_push<<<npeers * cpp, 512, 0, st[d]>>>((const uint4*)src[d], ds, cpp, bytes / 16);
        }
      };
      run();
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
      for (int it = 0; it < 5; ++it) run();
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e1[d], st[d])); }
      float worst = 0;
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventSynchronize(e1[d])); float ms; CK(cudaEventElapsedTime(&ms, e0[d], e1[d])); if (ms > worst) worst = ms; }
      const double egress = (double)bytes * npeers * 5 / (worst * 1e-3) / 1e9;
      printf("PUSH gpus=%d peers_each=%d ctas_per_peer=%2d total_ctas=%3d egress/GPU=%7.1f GB/s\n", n, npeers, cpp, cpp * npeers, egress);
      // pull variant: every GPU reads npeers peers' src buffers into its own dst
      auto runp = [&]() {
        for (int d = 0; d < n; ++d) {
          CK(cudaSetDevice(d));
          Srcs ss;
          for (int j = 0; j < npeers; ++j) { int p = (d + 1 + j) % n; ss.s[j] = (const uint4*)src[p]; }
          k_pull<<<npeers * cpp, 512, 0, st[d]>>>(ss, (uint4*)dst[d], cpp, bytes / 16);
        }
      };
      runp();
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
      for (int it = 0; it < 5; ++it) runp();
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e1[d], st[d])); }
      worst = 0;
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventSynchronize(e1[d])); float ms; CK(cudaEventElapsedTime(&ms, e0[d], e1[d])); if (ms > worst) worst = ms; }
      printf("PULL gpus=%d peers_each=%d ctas_per_peer=%2d total_ctas=%3d ingress/GPU=%7.1f GB/s\n", n, npeers, cpp, cpp * npeers, (double)bytes * npeers * 5 / (worst * 1e-3) / 1e9);
    }
  }
  return 0;
}
