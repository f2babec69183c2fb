// Tensor-core Gram-distance instantiations of the tcgen05 operator kernel
// (kv_tc_kernel.cu, template flag TG): same source, second translation unit.
#define GPK_KV_TC_TG 1
#include "kv_tc_kernel.cu"
