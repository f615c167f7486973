// plan2s.cuh — two-pass in-place rdFFT for n = 2048 (sm_100a): R = 64 scalar register blocks.
//
// Same stages as plan2 (the paper's radix-2 schedule, P:L225-266 forward, Eq. 7 P:L268-287 inverse),
// regrouped as n = R * M with R = 64, M = 32:
//  pass 1 (stages m = 1 .. 32): thread c owns ONE decimated subsequence x[c :: 32] (64 values, one
//    2-byte / 4-byte shared load each from the TMA-staged tile), runs rfft_fwd_reg<64> in registers
//    and writes window rev_5(c) (per-stage invariant, reading C5) with 16 128-bit stores;
//  last pass (stages m = 64 .. n/2): by Prop. 1 the groups close over S_k = {64 j +- k}; lane k
//    (k = 1 .. 32, one warp per vector) loads its 2 M scalars, applies W_n^{k rev_5(j)} and a 32-point
//    complex DIT (the radix-2 butterflies regrouped, exactly plan2's last pass), and stores its packed
//    outputs straight to HBM (a warp covers 32 consecutive slots of one row per store, as plan3's FD);
//    the block DCs (slots 64 j) form a real 32-point FFT on one lane per vector of the last warp.
// Against plan3 (three passes: R = 32, a 4-point middle pass, a 16-point last pass) this drops one
// shared-memory round trip of the fp32 intermediate per element and the middle pass's twiddles.
//
// Shared layout: plain fp32 slots (not plan2's half pairs — a thread holds one subsequence, not two),
// window w at base(w) = 68 w + 4 (w >> 3): the 4-float pad after every window holds the zero imaginary
// input of lane k = 32, and the extra 4 floats per 8 windows spread the 8 lanes of a 128-bit store
// phase (windows rev_5(c), c = 8t .. 8t + 7, whose low window bits agree) over 8 bank groups
// (conflict-free, checked by a bank simulation).  Row skew 4 floats per vector (the DC lanes).
// Last-pass twiddles W_n^{k r}, r = 4 a + b: table of W_n^{4 k a} (a < 8) times a per-lane
// W_n^{k b} (b < 4, registers), 2 KB instead of 8 KB of table (4 CTAs/SM instead of 3).
// Inverse: the last pass first, reading the staged bf16 / fp32 tile directly (plan2o's scheme), with
// conjugate twiddles and 1/n folded into the table; then pass 1 inverse, storing to HBM.
// Dispatched (2^20 vectors, fraction of measured HBM, gpurun_out r02_o): the bf16 forward with the
// output tile and 3 vectors per CTA (plan3 0.622 -> 0.706; without the tile 0.656) and the fp32
// inverse (plan3 0.916 -> 0.970).  The bf16 inverse (0.58-0.60: 64 two-byte stores per thread) and the
// fp32 forward (0.89-0.92) stay on plan3 (0.631 / 0.919).
#pragma once

#include "plan2.cuh"

namespace rdfft {

template <typename T, int N_, int VT_, bool O_ = false>
struct Plan2s {
  using elem = T;
  // O: the outputs (forward last pass + DC lanes, inverse pass 1) go to an output staging tile that one
  // thread stores with TMA bulk copies (plan2's rdfft2fo_kernel scheme) instead of 2- / 4-byte STGs
  static constexpr bool O = O_;
  static constexpr int N = N_, R = 64, LR = 6, M = N / R, LM = ilog2c<M>(), S = N / R, LS = ilog2c<S>();
  static constexpr int VT = VT_;
  static constexpr int NT = VT * 32;  // one warp per vector in both passes
  static constexpr int WP = R + 4;
  __host__ __device__ static constexpr int base(int w) { return w * WP + 4 * (w >> 3); }
  static constexpr int ROWA = ((base(S) + 28 + 15) / 16) * 16;
  __host__ __device__ static constexpr int skew(int v) { return 4 * (v & 7); }
  __host__ __device__ static constexpr int row(int v) { return v * ROWA + skew(v); }
  static constexpr int SROW = N + 16 / (int)sizeof(T);  // staged row (+16 B: DC lanes on distinct banks)
  static constexpr int STAGE = VT * SROW * (int)sizeof(T);
  static constexpr int TWL = (M / 4) * 32;  // W_n^{4 k a}, a < M/4, k = 1 .. 32
  static constexpr int OROW = O_ ? N + 16 / (int)sizeof(T) : 0;
  static_assert(S == 32 && M == 32, "plan2s shape: n = 2048");
  static_assert((SROW * (int)sizeof(T)) % 16 == 0 && ROWA % 4 == 0, "16-byte aligned rows");
};

template <typename P>
struct P2sSmem {  // [stage][O][H][TW][bar]
  static constexpr size_t O_OFF = (size_t)P::STAGE;
  static constexpr size_t H_OFF = O_OFF + (size_t)P::VT * P::OROW * sizeof(typename P::elem);
  static constexpr size_t TW_OFF = H_OFF + (size_t)(P::VT * P::ROWA + 16) * 4;
  static constexpr size_t BAR_OFF = TW_OFF + (size_t)P::TWL * 8;
  static constexpr size_t BYTES = BAR_OFF + 8;
};

// Last-pass twiddle of lane k: W^{k r} = h[(r >> 2) 32] * w[r & 3] (w[0] = 1).
struct STw {
  const float2* h;
  float2 w1, w2, w3;
  template <int R_>
  __device__ __forceinline__ float2 at() const {
    constexpr int a = R_ >> 2, b = R_ & 3;
    const float2 t = h[a * 32];
    if constexpr (b == 0) {
      return t;
    } else {
      const float2 w = b == 1 ? w1 : (b == 2 ? w2 : w3);
      return make_float2(fmaf(t.x, w.x, -t.y * w.y), fmaf(t.x, w.y, t.y * w.x));
    }
  }
};

template <typename P, bool kInv>
__global__ void __launch_bounds__(P::NT) rdfft2s_kernel(typename P::elem* __restrict__ x, int64_t batch) {
  using T = typename P::elem;
  using L = P2sSmem<P>;
  constexpr int VT = P::VT, N = P::N, R = P::R, M = P::M, LM = P::LM, S = P::S, NT = P::NT;
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  const T* stg = reinterpret_cast<const T*>(base);
  float* H = reinterpret_cast<float*>(base + L::H_OFF);
  T* O = reinterpret_cast<T*>(base + L::O_OFF);
  using STO = std::conditional_t<P::O, sst1<T>, gio<T>>;  // output stores: O tile or HBM
  float2* TW = reinterpret_cast<float2*>(base + L::TW_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  const int tid = threadIdx.x;
  // tables: TW[a 32 + k-1] = W_N^{4 k a} (inverse: conjugate / N)
  for (int e = tid; e < P::TWL; e += NT) {
    const int a = e / 32, k = 1 + e % 32;
    float s, c;
    sincospif(2.0f * (float)(4 * k * a) / (float)N, &s, &c);
    TW[e] = kInv ? make_float2(c * (1.0f / N), s * (1.0f / N)) : make_float2(c, -s);
  }
  for (int e = tid; e < VT * S; e += NT) {  // window pads: the zero imaginary input of lane k = R/2
    float* pad = H + P::row(e / S) + P::base(e % S) + R;
    *reinterpret_cast<float4*>(pad) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  // ---- roles: warp v = vector v of the tile; lane = subsequence c (pass 1) / set k - 1 (last pass)
  const int v = tid / 32, lane = tid % 32;
  const int c = lane, w1 = rev_bits<5>(lane);
  float* h1 = H + P::row(v) + P::base(w1);
  const int k = 1 + lane;
  const bool kz = (k == R / 2);
  float* ha = H + P::row(v) + k;                      // slot j R + k at ha + base(j)
  float* hm = H + P::row(v) + (R - k);                // slot j R + R - k
  const float* hz = kz ? H + P::row(v) + R : hm;      // imaginary input (k = R/2: the pads)
  STw tw;
  tw.h = TW + (k - 1);
  {
    float s1, c1, s2, c2, s3, c3;
    sincospif(2.0f * (float)k / (float)N, &s1, &c1);
    sincospif(4.0f * (float)k / (float)N, &s2, &c2);
    sincospif(6.0f * (float)k / (float)N, &s3, &c3);
    const float sg = kInv ? 1.0f : -1.0f;
    tw.w1 = make_float2(c1, sg * s1);
    tw.w2 = make_float2(c2, sg * s2);
    tw.w3 = make_float2(c3, sg * s3);
  }
  const int dv = tid - (NT - 32);  // DC set of vector dv: lane dv of the last warp
  const float* hd = H + P::row(dv < 0 ? 0 : dv);
  const uint32_t k65536 = kTwo16;
  const int64_t ntiles = (batch + VT - 1) / VT;
  auto tile_rows = [&](int64_t t) { return (int)(batch - t * VT < VT ? batch - t * VT : VT); };
  __syncthreads();
  if (tid == 0 && (int64_t)blockIdx.x < ntiles)
    stage_issue_rows<P>(x + (int64_t)blockIdx.x * VT * N, tile_rows(blockIdx.x), base, bar);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int nv = tile_rows(tile);
    T* xt = x + tile * VT * (int64_t)N;
    const int64_t nxt = tile + gridDim.x;
    mbar_wait(bar, it & 1);
    if (!kInv) {
      // ---- pass 1: subsequence c -> window rev(c)
      if (v < nv) {
        float b[R];
        const T* src = stg + v * P::SROW + c;
        ct::static_for<0, R>([&](auto I) {
          constexpr int i = decltype(I)::value;
          b[rev_bits<P::LR>(i)] = sio1<T>::ld(src + S * i, k65536);
        });
        rfft_fwd_reg<R>(b);
        ct::static_for<0, R / 4>([&](auto I) {
          constexpr int i = 4 * decltype(I)::value;
          *reinterpret_cast<float4*>(h1 + i) = make_float4(b[i], b[i + 1], b[i + 2], b[i + 3]);
        });
      }
      if (P::O && tid == 0) bulk_wait_read<0>();  // the previous tile's bulk store has read O
      __syncthreads();  // H complete; staging buffer consumed
      if (tid == 0 && nxt < ntiles) stage_issue_rows<P>(x + nxt * VT * (int64_t)N, tile_rows(nxt), base, bar);
      // ---- last pass: set S_k -> packed outputs straight to HBM
      if (v < nv) {
        float zr[M], zi[M];
        ct::static_for<0, M>([&](auto J) {
          constexpr int j = decltype(J)::value;
          zr[j] = ha[P::base(j)];
          zi[j] = hz[P::base(j)];
        });
        ct::static_for<1, M>([&](auto J) {
          constexpr int j = decltype(J)::value;
          const float2 t = tw.template at<rev_bits<LM>(j)>();
          const float q = zr[j];
          zr[j] = fmaf(q, t.x, -zi[j] * t.y);
          zi[j] = fmaf(q, t.y, zi[j] * t.x);
        });
        cfft_dit<M>(zr, zi);
        T* ob = P::O ? O + v * P::OROW : xt + v * N;
        T* da = ob + k;
        T* dm = ob + (R - k);
        ct::static_for<0, M / 2>([&](auto Q) {
          constexpr int q = decltype(Q)::value;
          STO::st1(da + q * R, zr[q]);
          STO::st1(da + q * R + N / 2, -zi[q + M / 2]);
          if (!kz) {
            STO::st1(dm + (M / 2 - 1 - q) * R, zr[q + M / 2]);
            STO::st1(dm + (M / 2 - 1 - q) * R + N / 2, zi[q]);
          }
        });
      }
      if (dv >= 0 && dv < nv) {  // block DCs: real M-point FFT (input already bit-reversed)
        float d[M];
        ct::static_for<0, M>([&](auto J) {
          constexpr int j = decltype(J)::value;
          d[j] = hd[P::base(j)];
        });
        rfft_fwd_reg<M>(d);
        T* dd = P::O ? O + dv * P::OROW : xt + dv * N;
        ct::static_for<0, M / 2>([&](auto J) {
          constexpr int j = decltype(J)::value;
          STO::st1(dd + j * R, d[j]);
          STO::st1(dd + j * R + N / 2, d[j + M / 2]);
        });
      }
      if constexpr (P::O) fence_proxy_async_smem();
    } else {
      // ---- inverse last pass, reading the staged tile (natural order)
      if (v < nv) {
        const T* sa = stg + v * P::SROW + k;
        const T* sm = stg + v * P::SROW + (R - k);
        float zr[M], zi[M];
        ct::static_for<0, M / 2>([&](auto Q) {
          constexpr int q = decltype(Q)::value;
          zr[rev_bits<LM>(q)] = sio1<T>::ld(sa + q * R, k65536);                          // Re Y[q]
          zi[rev_bits<LM>(q + M / 2)] = -sio1<T>::ld(sa + q * R + N / 2, k65536);         // Im Y[q + M/2]
          zr[rev_bits<LM>(q + M / 2)] = sio1<T>::ld(sm + (M / 2 - 1 - q) * R, k65536);    // Re Y[q + M/2]
          zi[rev_bits<LM>(q)] = sio1<T>::ld(sm + (M / 2 - 1 - q) * R + N / 2, k65536);    // Im Y[q]
        });
        cfft_dit<M, true>(zr, zi);
        ct::static_for<0, M>([&](auto J) {
          constexpr int j = decltype(J)::value;
          constexpr int rj = rev_bits<LM>(j);
          const float2 t = tw.template at<rj>();
          const float q = zr[rj];
          zr[rj] = fmaf(q, t.x, -zi[rj] * t.y);
          zi[rj] = fmaf(q, t.y, zi[rj] * t.x);
        });
        ct::static_for<0, M>([&](auto J) {
          constexpr int j = decltype(J)::value;
          constexpr int rj = rev_bits<LM>(j);
          ha[P::base(j)] = zr[rj];
          if (!kz) hm[P::base(j)] = zi[rj];  // k = R/2: imaginary part (zero up to rounding) dropped
        });
      }
      if (dv >= 0 && dv < nv) {
        const T* s = stg + dv * P::SROW;
        float d[M];
        ct::static_for<0, M / 2>([&](auto J) {
          constexpr int j = decltype(J)::value;
          d[j] = sio1<T>::ld(s + j * R, k65536);
          d[j + M / 2] = sio1<T>::ld(s + j * R + N / 2, k65536);
        });
        rfft_inv_reg<M>(d);
        float* hdw = H + P::row(dv);
        ct::static_for<0, M>([&](auto J) {
          constexpr int j = decltype(J)::value;
          hdw[P::base(j)] = d[j] * (1.0f / N);
        });
      }
      if (P::O && tid == 0) bulk_wait_read<0>();  // the previous tile's bulk store has read O
      __syncthreads();  // H complete; staging buffer consumed
      if (tid == 0 && nxt < ntiles) stage_issue_rows<P>(x + nxt * VT * (int64_t)N, tile_rows(nxt), base, bar);
      // ---- inverse pass 1: window rev(c) -> subsequence c in HBM
      if (v < nv) {
        float b[R];
        ct::static_for<0, R / 4>([&](auto I) {
          constexpr int i = 4 * decltype(I)::value;
          const float4 f = *reinterpret_cast<const float4*>(h1 + i);
          b[i] = f.x;
          b[i + 1] = f.y;
          b[i + 2] = f.z;
          b[i + 3] = f.w;
        });
        rfft_inv_reg<R>(b);
        T* dst = (P::O ? O + v * P::OROW : xt + v * N) + c;
        ct::static_for<0, R>([&](auto I) {
          constexpr int i = decltype(I)::value;
          STO::st1(dst + S * i, b[rev_bits<P::LR>(i)]);
        });
      }
      if constexpr (P::O) fence_proxy_async_smem();
    }
    __syncthreads();  // H free for the next tile (O complete)
    if constexpr (P::O) {
      if (tid == 0) {
        for (int vv = 0; vv < nv; ++vv) bulk_s2g(xt + (int64_t)vv * N, O + vv * P::OROW, (uint32_t)(N * sizeof(T)));
        bulk_commit();
      }
    }
  }
  if (P::O && tid == 0) bulk_wait<0>();
}

template <typename P, bool kInv>
bool launch_plan2s_dir(typename P::elem* x, int64_t batch, int sms, cudaStream_t st) {
  using L = P2sSmem<P>;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  auto k = rdfft2s_kernel<P, kInv>;
  static int per_sm_dev[kMaxDevices] = {};
  int& per_sm = per_sm_dev[device_index()];
  if (!per_sm) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, P::NT, L::BYTES);
    if (per_sm < 1) per_sm = 1;
    if (verbose())
      std::fprintf(stderr, "[rdfft] plan2s n=%d VT=%d O=%d inv=%d: %zu B smem, %d threads, %d CTAs/SM\n", P::N,
                   P::VT, (int)P::O, (int)kInv, (size_t)L::BYTES, P::NT, per_sm);
  }
  const int64_t tiles = (batch + P::VT - 1) / P::VT;
  const int grid = (int)(tiles < (int64_t)per_sm * sms ? tiles : (int64_t)per_sm * sms);
  k<<<grid, P::NT, L::BYTES, st>>>(x, batch);
  return true;
}

}  // namespace rdfft
