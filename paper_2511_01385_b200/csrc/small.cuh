// small.cuh — rdFFT for n <= 64 (bf16 n <= 128): one thread owns one vector.
//
// The whole transform is the paper's stage schedule (rfft_fwd_reg / rfft_inv_reg) on
// n registers with compile-time twiddles; the bit reversal is a compile-time register renaming.
// Each lane moves its own n-element row with 128-bit accesses: a warp instruction touches 32 rows,
// the rows' remaining 16-byte pieces come from L1 on the following instructions, so DRAM traffic
// stays one read and one write per element.
// Rows of >= 32 bytes instead go through a per-warp shared-memory transpose: the warp loads and stores
// its 32 rows with fully coalesced 512-byte instructions and each lane reads / writes its own row from
// shared memory (rows padded by 16 bytes: an odd number of 16-byte chunks per row, so a quarter-warp
// phase of own-row accesses hits 8 distinct 16-byte bank groups).  With per-lane rows a warp
// instruction touched 32 lines and L1 could not hold them (128-byte rows: 0.54 of HBM at any
// occupancy).  Measured (2^20 vectors, fraction of HBM, gpurun_out r02_x / r02_y): bf16 n = 16 / 32 /
// 64 0.70 / 0.81 / 0.54 -> 0.79 / 0.90 / 0.90; fp32 n = 16 / 32 0.80 / 0.52 -> 0.97 / 0.91; and it now
// also runs fp32 n = 64 (the two-pass plan's 0.80 / 0.60 -> 0.95 / 0.95) and bf16 n = 128 (0.64 / 0.60
// -> 0.82 / 0.86; 203 registers, no spills).
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
  constexpr bool kTr = (NV >= 2);              // rows of >= 32 bytes: shared-memory transpose (see header)
  constexpr int WARPS = kSmallThreads / 32;
  __shared__ uint4 tr[kTr ? WARPS : 1][kTr ? 32 : 1][kTr ? NV + 1 : 1];
  const int lane = threadIdx.x % 32, wq = threadIdx.x / 32;
  // kTr: the loop runs per warp over blocks of 32 consecutive rows (warp-uniform trip count)
  const int64_t first = kTr ? (blockIdx.x * (int64_t)kSmallThreads + wq * 32)
                            : (blockIdx.x * (int64_t)kSmallThreads + threadIdx.x);
  for (int64_t v0 = first; v0 < batch; v0 += (int64_t)gridDim.x * kSmallThreads) {
    const int64_t v = kTr ? v0 + lane : v0;
    T* row = x + v * N;
    float f[N];
    if constexpr (kTr) {
      const uint4* blk = reinterpret_cast<const uint4*>(x + v0 * N);
#pragma unroll
      for (int i = 0; i < NV; ++i) {  // 32 rows x 8 chunks, 512 contiguous bytes per instruction
        const int idx = 32 * i + lane, r = idx / NV, c = idx % NV;
        if (v0 + r < batch) tr[wq][r][c] = __ldcs(blk + idx);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < NV; ++i) io<T>::unpack16(tr[wq][lane][i], f + i * VEC);
    } else if constexpr (NV >= 1) {
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
    if constexpr (kTr) {
#pragma unroll
      for (int i = 0; i < NV; ++i) tr[wq][lane][i] = io<T>::pack16(f + i * VEC);
      __syncwarp();
      uint4* blk = reinterpret_cast<uint4*>(x + v0 * N);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int idx = 32 * i + lane, r = idx / NV, c = idx % NV;
        if (v0 + r < batch) __stcs(blk + idx, tr[wq][r][c]);
      }
      __syncwarp();  // tr is rewritten by the next block's loads
    } else if constexpr (NV >= 1) {
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
