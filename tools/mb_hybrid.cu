// Microbenchmark: does a copy engine add NVLink egress next to SM stores?
// Every GPU sends `bytes` to each of its N-1 peers at once:
//   sm      an SM kernel (128 CTAs, 16-byte stores) to all N-1 peers
//   hybrid  the copy engine to peer g+1 (cudaMemcpyPeerAsync) while the SM
//           kernel writes the other N-2 peers
//   ce      one copy-engine stream per peer
// Per-GPU egress GB/s, all GPUs in lock step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mb_hybrid tools/mb_hybrid.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                        \
  do {                                                               \
    cudaError_t e = (x);                                             \
    if (e != cudaSuccess) {                                          \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                 \
      exit(1);                                                       \
    }                                                                \
  } while (0)

struct Dst {
  char* p[8];
  int n;
};

__global__ void __launch_bounds__(256) k_push(const char* __restrict__ src, Dst d, long long bytes) {
  const int di = blockIdx.x % d.n;
  const int per = gridDim.x / d.n;
  const int bi = blockIdx.x / d.n;
  const long long nv = bytes / 16;
  const long long span = (nv + per - 1) / per;
  const long long lo = bi * span, hi = lo + span < nv ? lo + span : nv;
  uint4* dst = reinterpret_cast<uint4*>(d.p[di]);
  const uint4* s = reinterpret_cast<const uint4*>(src);
  constexpr int U = 4;
  for (long long i = lo + threadIdx.x; i < hi; i += (long long)blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + (long long)u * blockDim.x;
      if (j < hi) v[u] = s[j];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + (long long)u * blockDim.x;
      if (j < hi) dst[j] = v[u];
    }
  }
}

int main(int argc, char** argv) {
  const long long bytes = (argc > 1 ? atoll(argv[1]) : 256) << 20;
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 3) {
    printf("needs 3+ GPUs\n");
    return 0;
  }
  for (int a = 0; a < nd; ++a) {
    CK(cudaSetDevice(a));
    for (int b = 0; b < nd; ++b)
      if (a != b) cudaDeviceEnablePeerAccess(b, 0);
  }
  std::vector<char*> src(nd), dst(nd * nd);
  std::vector<std::vector<cudaStream_t>> st(nd, std::vector<cudaStream_t>(nd));
  for (int g = 0; g < nd; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMemset(src[g], 1, bytes));
    for (int h = 0; h < nd; ++h) {
      CK(cudaMalloc(&dst[g * nd + h], bytes));  // on g, written by h
      CK(cudaStreamCreateWithFlags(&st[g][h], cudaStreamNonBlocking));
    }
  }
  for (const char* mode : {"sm", "hybrid", "ce"}) {
    for (int ctas : {96, 128}) {
      auto launch = [&]() {
        for (int g = 0; g < nd; ++g) {
          CK(cudaSetDevice(g));
          Dst d{};
          const int succ = (g + 1) % nd;
          for (int h = 0; h < nd; ++h) {
            if (h == g) continue;
            const bool by_ce = mode[0] == 'c' || (mode[0] == 'h' && h == succ);
            if (by_ce)
              CK(cudaMemcpyPeerAsync(dst[h * nd + g], h, src[g], g, bytes, st[g][h]));
            else
              d.p[d.n++] = dst[h * nd + g];
          }
          if (d.n) k_push<<<ctas / d.n * d.n, 256, 0, st[g][g]>>>(src[g], d, bytes);
        }
        for (int g = 0; g < nd; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaDeviceSynchronize());
        }
      };
      launch();
      const int reps = 8;
      CK(cudaSetDevice(0));
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, 0));
      for (int r = 0; r < reps; ++r) launch();
      CK(cudaSetDevice(0));
      CK(cudaEventRecord(e1, 0));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("%-6s ctas=%3d N=%d: per-GPU egress %7.1f GB/s\n", mode, ctas, nd,
             (double)bytes * (nd - 1) * reps / (ms * 1e-3) / 1e9);
      if (mode[0] == 'c') break;
    }
  }
  return 0;
}
