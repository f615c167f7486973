// bca4.cuh — named barriers for the multi-pipe BCA kernels (bca5.cuh, bca_bwd5.cuh): one CTA per
// SM runs PIPES thread groups, each with its own H tile and its own named barrier, on disjoint token
// tiles.  A pipe waiting at its barrier leaves the SM to the other pipe, so barrier and latency
// stalls overlap as they would across independent CTAs, without a second copy of the W spectra.
#pragma once

#include "bca2.cuh"

namespace rdfft {

// bar.sync on a named barrier (ids 1..15; 0 is __syncthreads) for `nthreads` threads.
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace rdfft
