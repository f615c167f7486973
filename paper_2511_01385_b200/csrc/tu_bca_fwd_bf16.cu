// Explicit instantiation of the fused BCA forward launcher for __nv_bfloat16 (see fast.h).
#include "fast.h"
#include "bca5.cuh"
namespace rdfft {
template bool bca_fwd_fast<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, __nv_bfloat16*, int64_t, int, int, int, int, cudaStream_t, int, const float*);
}
