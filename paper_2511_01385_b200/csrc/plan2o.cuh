// plan2o.cuh — stand-alone bf16 inverse rdFFT with one shared-memory round trip fewer.
//
// Same two passes as plan2.cuh's inverse (the reversed graph, Eq. 7);
// only the data movement differs:
//  * the last pass reads its slots straight from the TMA-staged bf16 tile (one
//    2-byte load per slot) instead of first copying the tile into the fp32 half
//    pairs H (plan2's p2_load): 48 fewer shared-memory wavefronts per n = 1024
//    vector (the L1/shared pipe was the busiest unit, ~77 %);
//  * one extra warp runs the block-DC sets (real M-point FFTs) concurrently with
//    the last-pass warps.
// Measured (B200, 2^20 x 1024 bf16): 66.5 -> 75.5 % of HBM; n = 512: 63.7 -> 70 %.
// A forward counterpart (outputs packed to bf16 pairs in registers, emitted into
// an O tile over H after an extra barrier, de-interleaved with PRMT on the way
// out) measured slower (72 -> 67 %) and was dropped.
#pragma once

#include "plan2.cuh"

namespace rdfft {

template <int N_, int R_, int VT_, int NSTG_ = 1>
struct Plan2o : Plan2<__nv_bfloat16, N_, R_, VT_, NSTG_> {
  using B = Plan2<__nv_bfloat16, N_, R_, VT_, NSTG_>;
  static constexpr int DC0 = B::NT;          // the DC warp follows the last-pass warps
  static constexpr int NTT = B::NT + 32;     // threads per CTA
  // Staged rows 12 words (24 bf16) apart mod 32 banks: the interleaved vector pair of a last-pass
  // warp reads disjoint banks (8-9 words each), and so do the DC warp's 8 lanes (one per row).
  static constexpr int SROW = B::N + 24;
  static constexpr int STAGE = B::VT * SROW * 2;
};

__device__ __forceinline__ float bf16_at(const __nv_bfloat16* p, uint32_t k65536) {
  return __uint_as_float((uint32_t)(*reinterpret_cast<const unsigned short*>(p)) * k65536);
}

// inverse last pass reading the staged bf16 tile directly (same values p2_load + p2_last_inv read)
template <typename P>
__device__ __forceinline__ void p2o_last_inv(const P2Roles<P>& r, const __nv_bfloat16* st, int nv,
                                             uint32_t k65536) {
  constexpr int M = P::M, LM = P::LM, R = P::R, N = P::N;
  if (r.v2 < nv) {
    const __nv_bfloat16* sa = st + r.v2 * P::SROW + r.k;
    const __nv_bfloat16* sm = st + r.v2 * P::SROW + (R - r.k);
    float zr[M], zi[M];
    ct::static_for<0, M / 2>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      zr[rev_bits<LM>(q)] = bf16_at(sa + q * R, k65536);                              // Re Y[q]
      zi[rev_bits<LM>(q + M / 2)] = -bf16_at(sa + q * R + N / 2, k65536);             // Im Y[q + M/2]
      zr[rev_bits<LM>(q + M / 2)] = bf16_at(sm + (M / 2 - 1 - q) * R, k65536);        // Re Y[q + M/2]
      zi[rev_bits<LM>(q)] = bf16_at(sm + (M / 2 - 1 - q) * R + N / 2, k65536);        // Im Y[q]
    });
    cfft_dit<M, true>(zr, zi);
    ct::static_for<0, M / 2>([&](auto J2) {
      constexpr int j0 = 2 * decltype(J2)::value;
      constexpr int r0 = rev_bits<LM>(j0), r1 = rev_bits<LM>(j0 + 1);
      const float4 t2 = *reinterpret_cast<const float4*>(r.twi + j0);
      const float q0 = zr[r0];
      zr[r0] = fmaf(q0, t2.x, -zi[r0] * t2.y);
      zi[r0] = fmaf(q0, t2.y, zi[r0] * t2.x);
      const float q1 = zr[r1];
      zr[r1] = fmaf(q1, t2.z, -zi[r1] * t2.w);
      zi[r1] = fmaf(q1, t2.w, zi[r1] * t2.z);
    });
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      constexpr int r1 = rev_bits<LM>(jj), r2 = rev_bits<LM>(jj + M / 2);
      r.ha[jj * P::WSTR] = make_float2(zr[r1], zr[r2]);
      if (!r.kz) r.hm[jj * P::WSTR] = make_float2(zi[r1], zi[r2]);  // k = R/2: imaginary part dropped
    });
  }
}

template <typename P>
__device__ __forceinline__ void p2o_dc_inv(const P2Roles<P>& r, const __nv_bfloat16* st, int nv, uint32_t k65536) {
  constexpr int M = P::M, R = P::R, N = P::N;
  if (r.dv >= 0 && r.dv < nv) {
    const __nv_bfloat16* s = st + r.dv * P::SROW;
    float d[M];
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      d[jj] = bf16_at(s + jj * R, k65536);
      d[jj + M / 2] = bf16_at(s + jj * R + N / 2, k65536);
    });
    rfft_inv_reg<M>(d);
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      r.hd[jj * P::WSTR] = make_float2(d[jj] * (1.0f / N), d[jj + M / 2] * (1.0f / N));
    });
  }
}

template <typename P>
__global__ void __launch_bounds__(P::NTT, 4) rdfft2o_inv_kernel(__nv_bfloat16* __restrict__ x, int64_t batch) {
  using T = __nv_bfloat16;
  using L = P2Smem<P>;
  constexpr int VT = P::VT, N = P::N, NS = P::NSTG;
  static_assert(NS >= 1, "staged input");
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float2* H = reinterpret_cast<float2*>(base + L::H_OFF);
  float2* TW = reinterpret_cast<float2*>(base + L::TW_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  const int tid = threadIdx.x;
  p2_tables<P>(nullptr, TW, tid, P::NTT);
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) mbar_init(bar + q, 1);
    fence_mbar_init();
  }
  const P2Roles<P> r(H, TW, TW, tid);
  const uint32_t k65536 = kTwo16;
  // 32-bit tile indices (bf16 rows of n >= 128 elements: < 2^31 tiles in any device memory) keep
  // the loop state small enough for the 96-register cap of 4 CTAs/SM without spilling
  const int ntiles = (int)((batch + VT - 1) / VT);
  auto tile_rows = [&](int t) { return (int)(batch - (int64_t)t * VT < VT ? batch - (int64_t)t * VT : VT); };
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) {
      const int t = (int)blockIdx.x + q * (int)gridDim.x;
      if (t < ntiles) stage_issue_rows<P>(x + (int64_t)t * VT * N, tile_rows(t), base + q * P::STAGE, bar + q);
    }
  }
  const bool dcw = tid >= P::DC0;
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int nv = tile_rows(tile);
    T* xt = x + (int64_t)tile * VT * N;
    const int sb = it % NS;
    const T* st = reinterpret_cast<const T*>(base + sb * P::STAGE);
    const int nxt = tile + NS * (int)gridDim.x;
    mbar_wait(bar + sb, (it / NS) & 1);
    if (!dcw) p2o_last_inv<P>(r, st, nv, k65536);
    else p2o_dc_inv<P>(r, st, nv, k65536);
    __syncthreads();  // H complete; staging buffer consumed
    if (tid == 0 && nxt < ntiles)
      stage_issue_rows<P>(x + (int64_t)nxt * VT * N, tile_rows(nxt), base + sb * P::STAGE, bar + sb);
    p2_pass1_inv<P>(r, xt, nv);
    __syncthreads();  // H free for the next tile
  }
}

template <typename P>
bool launch_plan2o_inv(__nv_bfloat16* x, int64_t batch, int sms, cudaStream_t st) {
  using L = P2Smem<P>;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  auto k = rdfft2o_inv_kernel<P>;
  static int per_sm_dev[kMaxDevices] = {};
  int& per_sm = per_sm_dev[device_index()];
  if (!per_sm) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, P::NTT, L::BYTES);
    if (per_sm < 1) per_sm = 1;
    if (verbose())
      std::fprintf(stderr, "[rdfft] plan2o inverse n=%d R=%d VT=%d NSTG=%d: %zu B smem, %d threads, %d CTAs/SM\n",
                   P::N, P::R, P::VT, P::NSTG, (size_t)L::BYTES, P::NTT, per_sm);
  }
  const int64_t tiles = (batch + P::VT - 1) / P::VT;
  const int grid = (int)(tiles < (int64_t)per_sm * sms ? tiles : (int64_t)per_sm * sms);
  k<<<grid, P::NTT, L::BYTES, st>>>(x, batch);
  return true;
}

}  // namespace rdfft
