// Explicit instantiation of the fused BCA backward launcher for __nv_bfloat16 (see fast.h).
#include "fast.h"
#include "bca_bwd5.cuh"
namespace rdfft {
template bool bca_bwd_fast<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, const __nv_bfloat16*, __nv_bfloat16*, float*, int64_t, int, int, int, int,
                                 cudaStream_t, const float*);
}
