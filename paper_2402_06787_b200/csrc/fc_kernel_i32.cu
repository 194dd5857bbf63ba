// Instantiations of the forest kernel for FC_INT32 reductions (copies use the
// float32 table).  See fc_device.cuh.
#include "fc_device.cuh"

FC_DEFINE_KERNEL_TABLE(fc_kernel_ptr_i32, FC_INT32, false)
