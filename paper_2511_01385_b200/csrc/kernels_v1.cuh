// kernels_v1.cuh — straightforward shared-memory rdFFT kernels (one barrier per
// stage).  Correctness baseline and fallback for shapes the register-blocked
// kernels do not specialise; every entry still runs entirely on the GPU.
#pragma once

#include "stages.cuh"

namespace rdfft {

constexpr int kV1Threads = 256;
constexpr int kV1TileElems = 4096;  // fp32 elements of smem per tile

// One CTA transforms tiles of V = kV1TileElems / n vectors (grid-stride).
template <typename T, bool kInverse>
__global__ void __launch_bounds__(kV1Threads) rdfft_v1_kernel(T* __restrict__ x, int64_t batch, int n,
                                                                int logn) {
  __shared__ float s[kV1TileElems];
  __shared__ float2 tw[kMaxN / 2];
  make_twiddles(tw, n);
  const int V = kV1TileElems >> logn;
  const int64_t ntiles = (batch + V - 1) / V;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t v0 = tile * V;
    const int nv = (int)(batch - v0 < V ? batch - v0 : V);
    T* g = x + v0 * n;
    __syncthreads();  // twiddles ready / previous tile's smem reads done
    load_rows<T>(g, s, nv * n, n, logn, /*rev=*/!kInverse);
    __syncthreads();
    if (kInverse)
      inv_stages_smem(s, nv, n, logn, tw);
    else
      fwd_stages_smem(s, nv, n, logn, tw);
    store_rows<T>(g, s, nv * n, n, logn, /*rev=*/kInverse);
  }
}

// a <- a (.) b or a (.) conj(b) per bin; b broadcast when b_batch == 1.
template <typename T, bool kConj>
__global__ void __launch_bounds__(256) packed_mul_kernel(T* __restrict__ a, const T* __restrict__ b,
                                                         int64_t batch, int n, int logn, int64_t b_batch) {
  const int bins = (n >> 1);  // item k in [0, n/2): k = 0 handles slots 0 and n/2
  const int64_t items = batch * bins;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = it / bins;
    const int k = (int)(it - v * bins);
    T* ar = a + v * n;
    const T* br = b + (b_batch == 1 ? 0 : v) * n;
    if (k == 0) {
      io<T>::st(ar, io<T>::ld(ar) * io<T>::ld(br));
      if (n >= 2) io<T>::st(ar + bins, io<T>::ld(ar + bins) * io<T>::ld(br + bins));
    } else {
      const float2 A = make_float2(io<T>::ld(ar + k), io<T>::ld(ar + n - k));
      const float2 B = make_float2(io<T>::ld(br + k), io<T>::ld(br + n - k));
      const float2 C = kConj ? cmulc(A, B) : cmul(A, B);
      io<T>::st(ar + k, C.x);
      io<T>::st(ar + n - k, C.y);
    }
  }
}

}  // namespace rdfft
