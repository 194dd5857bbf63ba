// Microbenchmark: 128-bit vs 256-bit SM stores into peer memory over
// NVLink5/NVSwitch (sm_100 STG.E.ENL2.256).  One process drives every GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mb_v8 tools/mb_v8.cu
//   ./tools/bin/mb_v8 [MiB per destination]
// Patterns: uni (GPU0 -> GPU1), bidir (GPU0 <-> GPU1), a2a (every GPU to every
// other GPU, CTAs split over destinations); per-GPU egress GB/s.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                      \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

struct Dst {
  char* p[8];
  int n;
};

template <int W>  // bytes per lane per store: 16 or 32
__global__ void __launch_bounds__(256) k_push(const char* __restrict__ src, Dst d, long long bytes) {
  const int di = blockIdx.x % d.n;
  const int per = gridDim.x / d.n;
  const int bi = blockIdx.x / d.n;
  const long long nv = bytes / W;
  const long long span = (nv + per - 1) / per;
  const long long lo = bi * span, hi = lo + span < nv ? lo + span : nv;
  char* dst = d.p[di];
  constexpr int U = 4;
  for (long long i = lo + threadIdx.x; i < hi; i += (long long)blockDim.x * U) {
    if constexpr (W == 16) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = i + (long long)u * blockDim.x;
        if (j < hi) v[u] = reinterpret_cast<const uint4*>(src)[j];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = i + (long long)u * blockDim.x;
        if (j < hi) reinterpret_cast<uint4*>(dst)[j] = v[u];
      }
    } else {
      float a[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = i + (long long)u * blockDim.x;
        if (j < hi)
          asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=f"(a[u][0]), "=f"(a[u][1]), "=f"(a[u][2]), "=f"(a[u][3]), "=f"(a[u][4]),
                         "=f"(a[u][5]), "=f"(a[u][6]), "=f"(a[u][7])
                       : "l"(src + j * 32));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = i + (long long)u * blockDim.x;
        if (j < hi)
          asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + j * 32),
                       "f"(a[u][0]), "f"(a[u][1]), "f"(a[u][2]), "f"(a[u][3]), "f"(a[u][4]),
                       "f"(a[u][5]), "f"(a[u][6]), "f"(a[u][7])
                       : "memory");
      }
    }
  }
}

int main(int argc, char** argv) {
  const long long mib = argc > 1 ? atoll(argv[1]) : 256;
  const long long bytes = mib << 20;
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  for (int a = 0; a < nd; ++a) {
    CK(cudaSetDevice(a));
    for (int b = 0; b < nd; ++b)
      if (a != b) cudaDeviceEnablePeerAccess(b, 0);
  }
  std::vector<char*> src(nd), dst(nd * nd);
  std::vector<cudaStream_t> st(nd);
  for (int g = 0; g < nd; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMemset(src[g], 1, bytes));
    for (int h = 0; h < nd; ++h) CK(cudaMalloc(&dst[g * nd + h], bytes));  // dst[g][h]: on g, from h
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
  }
  const char* pats[] = {"uni", "bidir", "a2a"};
  for (int pi = 0; pi < 3; ++pi) {
    const int senders = pi == 0 ? 1 : (pi == 1 ? 2 : nd);
    for (int w : {16, 32}) {
      for (int ctas : {128, 148, 296}) {
        auto launch = [&]() {
          for (int g = 0; g < senders; ++g) {
            CK(cudaSetDevice(g));
            Dst d{};
            if (pi < 2) {
              d.n = 1;
              d.p[0] = dst[(1 - g) * nd + g];
            } else {
              d.n = 0;
              for (int h = 0; h < nd; ++h)
                if (h != g) d.p[d.n++] = dst[h * nd + g];
            }
            const int grid = ctas / d.n * d.n;
            if (w == 16)
              k_push<16><<<grid, 256, 0, st[g]>>>(src[g], d, bytes);
            else
              k_push<32><<<grid, 256, 0, st[g]>>>(src[g], d, bytes);
          }
        };
        launch();
        for (int g = 0; g < senders; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaStreamSynchronize(st[g]));
        }
        cudaEvent_t e0, e1;
        CK(cudaSetDevice(0));
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        const int reps = 10;
        CK(cudaEventRecord(e0, st[0]));
        for (int r = 0; r < reps; ++r) {
          launch();
          // keep the senders in lock step: every stream waits for all
          for (int g = 0; g < senders; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaStreamSynchronize(st[g]));
          }
        }
        CK(cudaSetDevice(0));
        CK(cudaEventRecord(e1, st[0]));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double per = (double)bytes * (pi == 2 ? (nd - 1) : 1) * reps / (ms * 1e-3) / 1e9;
        printf("%-5s W=%2d B/lane ctas=%3d: per-GPU egress %7.1f GB/s\n", pats[pi], w, ctas, per);
        CK(cudaEventDestroy(e0));
        CK(cudaEventDestroy(e1));
      }
    }
  }
  return 0;
}
