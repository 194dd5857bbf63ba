// Instantiations of the forest kernel for FC_FLOAT16 reductions (copies use the
// float32 table).  See fc_device.cuh.
#include "fc_device.cuh"

FC_DEFINE_KERNEL_TABLE(fc_kernel_ptr_f16, FC_FLOAT16, false)
