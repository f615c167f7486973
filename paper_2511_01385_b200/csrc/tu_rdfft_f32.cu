// Explicit instantiation of the rdFFT launchers for float (see fast.h).
#include "fast.h"
#include "plan3.cuh"
namespace rdfft {
template bool launch_rdfft_fast<float>(float*, int64_t, int, int, bool, int, cudaStream_t);
}
