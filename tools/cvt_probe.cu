// Probe: outputs of sm_100's cvt.rn.bf16x2.f32 for NaN, infinity, ties and
// denormals; these vectors pin oracle/forest_oracle.py::f32_to_bf16
// (tests/test_oracle.py::test_bf16_rounding_matches_sm100_cvt_vectors).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cvt_probe tools/cvt_probe.cu
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstring>
__global__ void k(const float* in, unsigned* out, int n) {
  int i = threadIdx.x;
  if (2 * i + 1 < n) {
    unsigned r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(in[2 * i + 1]), "f"(in[2 * i]));
    out[i] = r;
  }
}
int main() {
  unsigned bits[] = {0x7fc00000u, 0xffc00000u, 0x7f800001u, 0xff812345u, 0x7fa5a5a5u, 0x7f800000u, 0x3f808000u, 0x3f818000u, 0x00000001u, 0x807fffffu, 0x7f7fffffu, 0x3f80ffffu};
  const int n = 12;
  float h[n]; memcpy(h, bits, sizeof(bits));
  float* d; unsigned* o; cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, n / 2 * 4);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  k<<<1, 32>>>(d, o, n);
  unsigned r[n / 2]; cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  for (int i = 0; i < n / 2; ++i) printf("%08x -> %04x   %08x -> %04x\n", bits[2 * i], r[i] & 0xffff, bits[2 * i + 1], r[i] >> 16);
  return 0;
}
