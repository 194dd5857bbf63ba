// Microbenchmark: GPU-side gap between back-to-back launches of a ~10 us
// persistent-style kernel (128 CTAs x 256 threads) in a deep eager queue vs
// graph replay, for small (16 B) and large (~1.2 KB) __grid_constant__ params,
// with and without programmatic dependent launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_launch2 tools/mb_launch2.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int W> struct Par { long long spin_ns; long long pad[W]; };

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int W, int PDL>
__global__ void __launch_bounds__(256, 1) k_spin(const __grid_constant__ Par<W> p) {
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  const unsigned long long t0 = gt();
  while ((long long)(gt() - t0) < p.spin_ns) {}
  __syncthreads();
  if (PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int W, int PDL>
void run(cudaStream_t s, long long spin_ns, int smem = 0) {
  Par<W> p{}; p.spin_ns = spin_ns;
  auto launch = [&]() {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(128); cfg.blockDim = dim3(256); cfg.stream = s;
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = PDL;
    void* args[] = {(void*)&p};
    CK(cudaLaunchKernelExC(&cfg, (const void*)k_spin<W, PDL>, args));
  };
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  const int R = 2000;
  for (int i = 0; i < 50; ++i) launch();
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < R; ++i) launch();
  CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
  float ms_e; CK(cudaEventElapsedTime(&ms_e, a, b));
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < 200; ++i) launch();
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < R / 200; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
  float ms_g; CK(cudaEventElapsedTime(&ms_g, a, b));
  printf("smem %6d params %5zu B pdl=%d spin %5lld ns: eager %.2f us/launch (gap %.2f), graph %.2f (gap %.2f)\n",
         smem, sizeof(Par<W>), PDL, spin_ns, ms_e * 1e3 / R, ms_e * 1e3 / R - spin_ns * 1e-3,
         ms_g * 1e3 / R, ms_g * 1e3 / R - spin_ns * 1e-3);
  CK(cudaGraphExecDestroy(ge)); CK(cudaGraphDestroy(g));
}

int main() {
  CK(cudaSetDevice(0));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaFuncSetAttribute((const void*)k_spin<150, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10));
  CK(cudaFuncSetAttribute((const void*)k_spin<150, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10));
  for (long long ns : {2000LL, 10000LL}) {
    run<1, 0>(s, ns); run<1, 1>(s, ns);
    run<150, 0>(s, ns); run<150, 1>(s, ns);
    run<150, 0>(s, ns, 200 << 10); run<150, 1>(s, ns, 200 << 10);
  }
  return 0;
}
