// small.cuh — rdFFT for n <= 64: one thread owns one vector.
//
// The whole transform is the paper's stage schedule (rfft_fwd_reg / rfft_inv_reg) on
// n registers with compile-time twiddles; the bit reversal is a compile-time register renaming.
// Each lane moves its own n-element row with 128-bit accesses: a warp instruction touches 32 rows,
// the rows' remaining 16-byte pieces come from L1 on the following instructions, so DRAM traffic
// stays one read and one write per element.
#pragma once

#include "common.cuh"
#include "regfft.cuh"

namespace rdfft {

constexpr int kSmallThreads = 128;

template <typename T, int N, bool kInv>
__global__ void __launch_bounds__(kSmallThreads) rdfft_small_kernel(T* __restrict__ x, int64_t batch) {
  constexpr int VEC = io<T>::kVec;             // elements per 16-byte access
  constexpr int NV = N / VEC;                  // 16-byte accesses per row
  constexpr int LN = ilog2c<N>();
  for (int64_t v = blockIdx.x * (int64_t)kSmallThreads + threadIdx.x; v < batch;
       v += (int64_t)gridDim.x * kSmallThreads) {
    T* row = x + v * N;
    float f[N];
    if constexpr (NV >= 1) {
      uint4 u[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) u[i] = reinterpret_cast<const uint4*>(row)[i];
#pragma unroll
      for (int i = 0; i < NV; ++i) io<T>::unpack16(u[i], f + i * VEC);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) f[i] = io<T>::ld(row + i);
    }
    float b[N];
    if constexpr (!kInv) {
      ct::static_for<0, N>([&](auto I) {
        constexpr int i = decltype(I)::value;
        b[rev_bits<LN>(i)] = f[i];
      });
      rfft_fwd_reg<N>(b);
      ct::static_for<0, N>([&](auto I) {
        constexpr int i = decltype(I)::value;
        f[i] = b[i];
      });
    } else {
      ct::static_for<0, N>([&](auto I) {
        constexpr int i = decltype(I)::value;
        b[i] = f[i];
      });
      rfft_inv_reg<N>(b);  // N x (bit-reversed signal)
      ct::static_for<0, N>([&](auto I) {
        constexpr int i = decltype(I)::value;
        f[i] = b[rev_bits<LN>(i)] * (1.0f / N);
      });
    }
    if constexpr (NV >= 1) {
#pragma unroll
      for (int i = 0; i < NV; ++i) reinterpret_cast<uint4*>(row)[i] = io<T>::pack16(f + i * VEC);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) io<T>::st(row + i, f[i]);
    }
  }
}

template <typename T, int N>
bool launch_small(T* x, int64_t batch, bool inverse, int sms, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  const int64_t blocks = (batch + kSmallThreads - 1) / kSmallThreads;
  const int grid = (int)(blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16);
  if (inverse)
    rdfft_small_kernel<T, N, true><<<grid, kSmallThreads, 0, st>>>(x, batch);
  else
    rdfft_small_kernel<T, N, false><<<grid, kSmallThreads, 0, st>>>(x, batch);
  return true;
}

}  // namespace rdfft
