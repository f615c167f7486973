// Explicit instantiation of the fused BCA backward launcher for float (see fast.h).
#include "fast.h"
#include "bca_bwd5.cuh"
namespace rdfft {
template bool bca_bwd_fast<float>(const float*, const float*, const float*, float*, float*, int64_t, int, int, int, int,
                                 cudaStream_t, const float*);
}
