// Microbenchmark: back-to-back launch cost of a persistent-kernel-shaped
// grid (128 CTAs x 256 threads, ~1.2 KB of __grid_constant__ params), eager
// stream launches vs CUDA-graph replay, with and without PDL.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_launch tools/mb_launch.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

struct Big { long long w[150]; };
struct Ctl { unsigned done, epoch; };

template <int PDL>
__global__ void __launch_bounds__(256, 1) k_exit(const __grid_constant__ Big p, Ctl* ctl) {
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  if (PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(&ctl->done, 1u);
    if (prev == gridDim.x - 1) { ctl->done = 0; __threadfence(); atomicAdd(&ctl->epoch, (unsigned)p.w[0]); }
  }
}

// the same without fences (the kernel boundary orders the next launch)
template <int PDL>
__global__ void __launch_bounds__(256, 1) k_exit_nf(const __grid_constant__ Big p, Ctl* ctl) {
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  if (PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(&ctl->done, 1u);
    if (prev == gridDim.x - 1) { ctl->done = 0; ctl->epoch += (unsigned)p.w[0]; }
  }
}

template <int PDL>
__global__ void __launch_bounds__(256, 1) k_empty(const __grid_constant__ Big p, Ctl* ctl) {
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.w[1] == 12345) ctl->epoch = 0;
}

int main() {
  CK(cudaSetDevice(0));
  Ctl* ctl; CK(cudaMalloc(&ctl, sizeof(Ctl))); CK(cudaMemset(ctl, 0, sizeof(Ctl)));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  Big p{}; p.w[0] = 1;
  const int R = 1000;
  for (int grid : {16, 128, 148}) {
    for (int which = 0; which < 6; ++which) {
      const void* fn = which == 0 ? (const void*)k_empty<0> : which == 1 ? (const void*)k_empty<1>
                     : which == 2 ? (const void*)k_exit<0> : which == 3 ? (const void*)k_exit<1>
                     : which == 4 ? (const void*)k_exit_nf<0> : (const void*)k_exit_nf<1>;
      const int pdl = which & 1;
      auto launch = [&]() {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = pdl;
        void* args[] = {(void*)&p, (void*)&ctl};
        CK(cudaLaunchKernelExC(&cfg, fn, args));
      };
      for (int i = 0; i < 50; ++i) launch();
      CK(cudaStreamSynchronize(s));
      CK(cudaEventRecord(a, s));
      for (int i = 0; i < R; ++i) launch();
      CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
      float ms_e; CK(cudaEventElapsedTime(&ms_e, a, b));
      cudaGraph_t g; cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
      for (int i = 0; i < 100; ++i) launch();
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
      CK(cudaEventRecord(a, s));
      for (int i = 0; i < R / 100; ++i) CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
      float ms_g; CK(cudaEventElapsedTime(&ms_g, a, b));
      printf("grid %3d %-10s pdl=%d: eager %.2f us/launch, graph %.2f us/launch\n", grid,
             which < 2 ? "empty" : which < 4 ? "exit-count" : "exit-nofence", pdl, ms_e * 1e3 / R, ms_g * 1e3 / R);
      CK(cudaGraphExecDestroy(ge)); CK(cudaGraphDestroy(g));
    }
  }
  return 0;
}
