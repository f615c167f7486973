// Explicit instantiation of the rdFFT launchers for __nv_bfloat16 (see fast.h).
#include "fast.h"
#include "plan3.cuh"
namespace rdfft {
template bool launch_rdfft_fast<__nv_bfloat16>(__nv_bfloat16*, int64_t, int, int, bool, int, cudaStream_t);
}
