// Instantiations of the forest kernel for FC_FLOAT32 reductions (copies use the
// float32 table).  See fc_device.cuh.
#include "fc_device.cuh"

FC_DEFINE_KERNEL_TABLE(fc_kernel_ptr_f32, FC_FLOAT32, false)
