// Kernel selection and launch (host side of the kernel TUs).
#include <cuda_runtime.h>

#include "fc_internal.h"

#define FC_WPC 8
#define FC_BLOCK (32 * FC_WPC)
#define FC_SMEM_BYTES (8 * 3 * 8 * 1024)

const void* fc_kernel_ptr_f32(int ww, int proto);
const void* fc_kernel_ptr_bf16(int ww, int proto);
const void* fc_kernel_ptr_f16(int ww, int proto);
const void* fc_kernel_ptr_i32(int ww, int proto);
const void* fc_kernel_ptr_f32_avg(int ww, int proto);
const void* fc_kernel_ptr_bf16_avg(int ww, int proto);
const void* fc_kernel_ptr_f16_avg(int ww, int proto);

namespace {

const void* kernel_for(int rd, int ww, int proto, bool avg) {
  switch (rd) {
    case FC_BFLOAT16: return avg ? fc_kernel_ptr_bf16_avg(ww, proto) : fc_kernel_ptr_bf16(ww, proto);
    case FC_FLOAT16: return avg ? fc_kernel_ptr_f16_avg(ww, proto) : fc_kernel_ptr_f16(ww, proto);
    case FC_INT32: return fc_kernel_ptr_i32(ww, proto);  // AVG rejected for integers
    default: return avg ? fc_kernel_ptr_f32_avg(ww, proto) : fc_kernel_ptr_f32(ww, proto);
  }
}

int smem_for(int proto) { return proto ? 0 : FC_SMEM_BYTES; }  // LL128 keeps no smem ring

int ensure_smem_attr(const void* fn) {
  static const void* done[128] = {};
  for (auto& d : done) {
    if (d == fn) return 0;
    if (!d) {
      const cudaError_t e =
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, FC_SMEM_BYTES);
      if (e != cudaSuccess) return (int)e;
      d = fn;
      return 0;
    }
  }
  return 0;
}

}  // namespace

int fc_launch(const FcParams& p, int reduce_dtype, int cooperative, void* stream, int* grid_out) {
  const dim3 grid(p.nlocal * p.ctas_per_rank), block(FC_BLOCK);
  void* args[] = {(void*)&p};
  const void* fn = kernel_for(reduce_dtype, p.worker_warps, p.proto, p.op == FC_AVG);
  if (grid_out) *grid_out = (int)grid.x;
  const int a = ensure_smem_attr(fn);
  if (a) return a;
  cudaError_t err;
  const int smem = smem_for(p.proto);
  if (cooperative) {
    err = cudaLaunchCooperativeKernel(fn, grid, block, args, smem, (cudaStream_t)stream);
  } else if (p.pdl) {
    // programmatic dependent launch: overlap this launch with the tail of
    // the previous kernel in the stream (the kernel waits in its prologue)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    err = cudaLaunchKernelExC(&cfg, fn, args);
  } else {
    err = cudaLaunchKernel(fn, grid, block, args, smem, (cudaStream_t)stream);
  }
  return (int)err;
}

int fc_max_ctas_per_sm(int reduce_dtype, int* out) {
  int best = 1 << 30;
  for (int proto = 0; proto < 2; ++proto) {
    const void* fn = kernel_for(reduce_dtype, 8, proto, false);
    const int a = ensure_smem_attr(fn);
    if (a) return a;
    int v = 0;
    const cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, FC_BLOCK, FC_SMEM_BYTES);
    if (e != cudaSuccess) return (int)e;
    if (v < best) best = v;
  }
  *out = best;
  return 0;
}

int fc_warps_per_cta() { return FC_WPC; }
