// Instantiations of the forest kernel for FC_BFLOAT16 reductions with op AVG (the
// tree roots scale their fp32 sum by 1/N before the final rounding).  Kept
// apart from the SUM kernels so those carry no extra register pressure.
#include "fc_device.cuh"

FC_DEFINE_KERNEL_TABLE(fc_kernel_ptr_bf16_avg, FC_BFLOAT16, true)
