// Explicit instantiation of the fused BCA forward launcher for float (see fast.h).
#include "fast.h"
#include "bca5.cuh"
namespace rdfft {
template bool bca_fwd_fast<float>(const float*, const float*, float*, int64_t, int, int, int, int, cudaStream_t, int, const float*);
}
