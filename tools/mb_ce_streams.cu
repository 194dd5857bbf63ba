// Microbenchmark: does splitting one peer transfer over several streams
// (several copy engines) raise NVLink egress past one copy engine's rate?
// GPU0 <-> GPU1 both sending `MiB` at once, the transfer cut into k equal
// pieces issued on k streams (k = 1, 2, 4, 8); per-GPU egress GB/s.  With 4+
// GPUs also the all-to-all pattern (every GPU to every peer) with k streams
// per peer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mb_ce_streams tools/mb_ce_streams.cu
//   ./tools/bin/mb_ce_streams [MiB]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                \
  do {                                                       \
    cudaError_t e = (x);                                     \
    if (e != cudaSuccess) {                                  \
      printf("%s: %s\n", #x, cudaGetErrorString(e));         \
      exit(1);                                               \
    }                                                        \
  } while (0)

int main(int argc, char** argv) {
  const long long bytes = (argc > 1 ? atoll(argv[1]) : 512) << 20;
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
  const int KMAX = 8;
  std::vector<char*> src(nd), dst(nd * nd);
  std::vector<std::vector<cudaStream_t>> st(nd, std::vector<cudaStream_t>(nd * KMAX));
  for (int g = 0; g < nd; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMemset(src[g], 1, bytes));
    for (int h = 0; h < nd; ++h) CK(cudaMalloc(&dst[g * nd + h], bytes));  // on g, from h
    for (auto& s : st[g]) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  for (int pat = 0; pat < (nd >= 4 ? 2 : 1); ++pat) {
    const int ng = pat == 0 ? 2 : nd;
    for (int k : {1, 2, 4, 8}) {
      auto launch = [&]() {
        for (int g = 0; g < ng; ++g) {
          CK(cudaSetDevice(g));
          int si = 0;
          for (int h = 0; h < ng; ++h) {
            if (h == g) continue;
            const long long piece = bytes / k;
            for (int p = 0; p < k; ++p)
              CK(cudaMemcpyAsync(dst[h * nd + g] + p * piece, src[g] + p * piece, piece,
                                 cudaMemcpyDeviceToDevice, st[g][si++]));
          }
        }
        for (int g = 0; g < ng; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaDeviceSynchronize());
        }
      };
      launch();
      const int reps = 6;
      // device time on GPU 0 over reps (every rep synchronises all GPUs)
      CK(cudaSetDevice(0));
      cudaEvent_t w0, w1;
      CK(cudaEventCreateWithFlags(&w0, cudaEventDefault));
      CK(cudaEventCreateWithFlags(&w1, cudaEventDefault));
      CK(cudaEventRecord(w0, 0));
      for (int r = 0; r < reps; ++r) launch();
      CK(cudaSetDevice(0));
      CK(cudaEventRecord(w1, 0));
      CK(cudaEventSynchronize(w1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, w0, w1));
      printf("%-8s k=%d streams per peer: per-GPU egress %7.1f GB/s\n", pat == 0 ? "pair" : "all2all", k,
             (double)bytes * (ng - 1) * reps / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
