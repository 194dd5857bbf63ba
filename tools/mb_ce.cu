// Microbenchmark: copy-engine (cudaMemcpyPeerAsync) vs SM-store bandwidth over
// NVLink5/NVSwitch, one process driving every GPU of the box.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_ce tools/mb_ce.cu
//   ./mb_ce [MiB per transfer]
// Patterns (per-GPU egress GB/s reported):
//   uni   GPU0 -> GPU1
//   bidir GPU0 <-> GPU1
//   a2a   every GPU -> every other GPU at once (one stream per destination)
// each with copy engines ("ce"), an SM kernel ("sm", 128 CTAs of 16-byte
// stores split over the destinations), and both at once ("ce+sm": half the
// bytes each).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

struct Dst { uint4* p[8]; int n; };

__global__ void k_push(const uint4* __restrict__ src, Dst d, long long nvec) {
  // CTA b serves destination b % n; per destination the CTAs split the range
  const int di = blockIdx.x % d.n;
  const int per = gridDim.x / d.n;
  const int bi = blockIdx.x / d.n;
  const long long span = (nvec + per - 1) / per;
  const long long lo = bi * span, hi = lo + span < nvec ? lo + span : nvec;
  uint4* dst = d.p[di];
  constexpr int U = 8;
  for (long long i = lo + threadIdx.x; i < hi; i += (long long)blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = i + (long long)u * blockDim.x; if (j < hi) v[u] = __ldcg(src + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = i + (long long)u * blockDim.x; if (j < hi) dst[j] = v[u]; }
  }
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)(argc > 1 ? atoll(argv[1]) : 256) << 20;
  int nd; CK(cudaGetDeviceCount(&nd));
  if (nd < 2) { printf("need >= 2 GPUs\n"); return 0; }
  std::vector<char*> src(nd), dst(nd * nd);
  std::vector<cudaStream_t> st(nd * nd);
  std::vector<cudaEvent_t> e0(nd), e1(nd);
  for (int g = 0; g < nd; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < nd; ++h) if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMemset(src[g], g + 1, bytes));
    for (int h = 0; h < nd; ++h) { CK(cudaMalloc(&dst[g * nd + h], bytes)); CK(cudaStreamCreateWithFlags(&st[g * nd + h], cudaStreamNonBlocking)); }
    CK(cudaEventCreate(&e0[g])); CK(cudaEventCreate(&e1[g]));
  }
  // dst[h*nd+g]: buffer on GPU h receiving from g
  auto run = [&](const char* pat, int mode, int reps) {
    // senders and their destinations
    std::vector<std::vector<int>> to(nd);
    if (!strcmp(pat, "uni")) to[0] = {1};
    else if (!strcmp(pat, "bidir")) { to[0] = {1}; to[1] = {0}; }
    else for (int g = 0; g < nd; ++g) for (int h = 0; h < nd; ++h) if (h != g) to[g].push_back(h);
    for (int g = 0; g < nd; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
    float worst = 0; double egress = 0;
    for (int it = -1; it < reps; ++it) {
      for (int g = 0; g < nd; ++g) {
        if (to[g].empty()) continue;
        CK(cudaSetDevice(g));
        cudaStream_t s0 = st[g * nd + g];
        CK(cudaEventRecord(e0[g], s0));
        const size_t sm_bytes = mode == 0 ? 0 : mode == 1 ? bytes : bytes / 2;
        const size_t ce_bytes = bytes - sm_bytes;
        for (int h : to[g]) {
          cudaStream_t s = st[g * nd + h];
          CK(cudaStreamWaitEvent(s, e0[g], 0));
          if (ce_bytes) CK(cudaMemcpyPeerAsync(dst[h * nd + g], h, src[g], g, ce_bytes, s));
        }
        if (sm_bytes) {
          Dst d; d.n = (int)to[g].size();
          for (int i = 0; i < d.n; ++i) d.p[i] = (uint4*)(dst[to[g][i] * nd + g] + ce_bytes);
          const int ctas = 128 / d.n * d.n;
          k_push<<<ctas, 512, 0, s0>>>((const uint4*)(src[g] + ce_bytes), d, (long long)(sm_bytes / 16));
        }
        for (int h : to[g]) {
          cudaEvent_t ev; CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          CK(cudaEventRecord(ev, st[g * nd + h])); CK(cudaStreamWaitEvent(s0, ev, 0)); CK(cudaEventDestroy(ev));
        }
        CK(cudaEventRecord(e1[g], s0));
      }
      for (int g = 0; g < nd; ++g) if (!to[g].empty()) { CK(cudaSetDevice(g)); CK(cudaEventSynchronize(e1[g])); }
      if (it < 0) continue;
      for (int g = 0; g < nd; ++g) {
        if (to[g].empty()) continue;
        float ms; CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        if (ms > worst) worst = ms;
      }
      egress = (double)bytes * to[0].size();
    }
    (void)worst;
    // report the last rep's slowest sender
    printf("%-6s %-6s: per-GPU egress %7.1f GB/s (%zu MiB x %zu dst, %.3f ms)\n", pat,
           mode == 0 ? "ce" : mode == 1 ? "sm" : "ce+sm", egress / (worst * 1e-3) / 1e9,
           bytes >> 20, to[0].size(), worst);
  };
  for (const char* pat : {"uni", "bidir", "a2a"})
    for (int mode = 0; mode < 3; ++mode) run(pat, mode, 5);
  return 0;
}
