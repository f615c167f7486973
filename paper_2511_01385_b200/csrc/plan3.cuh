// plan3.cuh — three-pass register-blocked rdFFT for n = 2048, 4096 (sm_100a).
//
// n = R * M2 * M3 with R = 32 (pass 1, the paper's first 5 stages per decimated
// subsequence, exactly as plan2), M2 = 4 (middle pass: stages m = 32, 64 on the
// closed sets S_k = {j 32 +- k} of each 128-slot window, both half-pair windows
// in the two float2 lanes), M3 = n / 128 (last pass: stages m = 128 .. n/2 on
// S_k = {j 128 +- k}, k = 1 .. 64).  Every pass is the paper's radix-2 stages
// regrouped as "twiddle + small complex DIT FFT" on a Prop. 1 closed set; the
// block DCs of each pass form a real FFT run by dedicated lanes.  The shared
// layout (padded 32-slot windows, half pairs, row skew) is plan2's.
// The forward's last pass stores its outputs straight to HBM (Plan3::FD: a warp covers 32
// consecutive slots of one row per 2-byte / 4-byte store), which drops the H -> HBM store phase
// and one barrier: bf16 n = 2048 fwd 0.55 -> 0.59 of HBM, 4096 0.50 -> 0.53, fp32 2048
// 0.81 -> 0.88, 4096 0.72 -> 0.74 (profiles/r01_v13_sweep.jsonl).
// NSTG = 0 (pass 1 / the inverse's first pass reading HBM directly, 5 CTAs/SM instead of 4) is
// supported but measured slower for every (n, dtype): bf16 4096 0.53 -> 0.47, fp32 2048 0.92 -> 0.69.
#pragma once

#include "plan2.cuh"
#include "plan2o.cuh"
#include "small.cuh"
#include "planl.cuh"
#include "plan2s.cuh"

namespace rdfft {

template <typename T, int N_, int VT_, int NSTG_ = 2, bool FD_ = false>
struct Plan3 {
  using elem = T;
  static constexpr int N = N_, VT = VT_, R = 32, NSTG = NSTG_;
  static constexpr bool FD = FD_;  // forward last pass stores straight to HBM (see Plan2::FD)
  static constexpr int M2 = 4, W2 = 128;     // middle pass
  static constexpr int M3 = N / W2, LM3 = ilog2c<M3>();
  static constexpr int LR = 5, S = N / R, LS = ilog2c<S>(), P1 = S / 2;
  static constexpr int NT = VT * P1;
  static constexpr int WSTR = R + 2;
  static constexpr int NWIN = S / 2;
  static constexpr int ROWA = ((NWIN * WSTR + 14 + 15) / 16) * 16;
  static constexpr int HF = VT * ROWA + 16;
  static constexpr int KM = R / 2;           // middle-pass lanes per window (k = 1 .. 16)
  static constexpr int WPV = N / (2 * W2);   // middle-pass windows per vector (first half)
  static constexpr int MIPV = WPV * KM;      // middle general items per vector
  static constexpr int KL = W2 / 2;          // last-pass lanes per vector (k = 1 .. 64)
  // last-pass twiddles W_N^{k r}, r = rev(j) = 4a + b: table of W_N^{4 k a} (a < M3/4), times W_N^{k b}
  // (b < 4) held in registers -> 4 KB instead of 16 KB at n = 4096 (4 CTAs/SM instead of 3)
  static constexpr int TWM = M2 * KM, TWL = (M3 / 4) * KL;
  static constexpr int CHV = N / 4;
  static constexpr int STAGE = VT * N * (int)sizeof(T);
  static_assert(M3 >= 4 && M3 <= 32, "plan3 shape");
  static_assert(NT % 32 == 0 && (NT % MIPV == 0 || MIPV % NT == 0) && (VT * KL) % NT == 0 && CHV % NT == 0,
                "plan3 mapping");
  static_assert(VT <= 8, "compile-time skew offsets assume v < 8");
  __host__ __device__ static constexpr int skew(int v) { return 2 * (v & 7); }
  __host__ __device__ static constexpr int row(int v) { return v * ROWA + skew(v); }
  // physical float2 offset (within a row) of logical half-pair index q
  __host__ __device__ static constexpr int pos(int q) { return (q / R) * WSTR + (q % R); }
};

template <typename P>
struct P3Smem {  // [stage 0][stage 1][H][TWm][TWl][bars]
  static constexpr size_t H_OFF = (size_t)P::NSTG * P::STAGE;
  static constexpr size_t TWM_OFF = H_OFF + (size_t)P::HF * 8;
  static constexpr size_t TWL_OFF = TWM_OFF + (size_t)P::TWM * 8;
  static constexpr size_t BAR_OFF = TWL_OFF + (size_t)P::TWL * 8;
  static constexpr size_t BYTES = BAR_OFF + 8 * (P::NSTG > 0 ? P::NSTG : 1);
};

// Middle-pass general set on both half-pair lanes: Z_j(k), j < 4, of one 128-slot window.
template <bool kInv>
__device__ __forceinline__ void p3_mid_set(float2* ha, float2* hm, const float2* hmi, float2* hmo, const float2* tw) {
  constexpr int M = 4, WS = 34;
  float zr[2][M], zi[2][M];
  if (!kInv) {
    ct::static_for<0, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 a = ha[j * WS], b = hmi[j * WS];
      zr[0][j] = a.x; zr[1][j] = a.y;
      zi[0][j] = b.x; zi[1][j] = b.y;
    });
    ct::static_for<1, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 t = tw[j * 16];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float q = zr[h][j];
        zr[h][j] = fmaf(q, t.x, -zi[h][j] * t.y);
        zi[h][j] = fmaf(q, t.y, zi[h][j] * t.x);
      }
    });
    cfft_dit<M>(zr[0], zi[0]);
    cfft_dit<M>(zr[1], zi[1]);
    // asc[q] <- q < 2 ? Re Y[q] : -Im Y[q];  mirror[3 - q] <- q < 2 ? Im Y[q] : Re Y[q]
    ct::static_for<0, M>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      if constexpr (q < M / 2) {
        ha[q * WS] = make_float2(zr[0][q], zr[1][q]);
        hm[(M - 1 - q) * WS] = make_float2(zi[0][q], zi[1][q]);
      } else {
        ha[q * WS] = make_float2(-zi[0][q], -zi[1][q]);
        hm[(M - 1 - q) * WS] = make_float2(zr[0][q], zr[1][q]);
      }
    });
  } else {
    // Y[q] from the packed window; load into register rev(q) for the conjugate DIT pass
    ct::static_for<0, M>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int rq = rev_bits<2>(q);
      const float2 a = ha[q * WS], b = hm[(M - 1 - q) * WS];
      if constexpr (q < M / 2) {
        zr[0][rq] = a.x; zr[1][rq] = a.y;
        zi[0][rq] = b.x; zi[1][rq] = b.y;
      } else {
        zi[0][rq] = -a.x; zi[1][rq] = -a.y;
        zr[0][rq] = b.x; zr[1][rq] = b.y;
      }
    });
    cfft_dit<M, true>(zr[0], zi[0]);
    cfft_dit<M, true>(zr[1], zi[1]);
    ct::static_for<0, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      constexpr int rj = rev_bits<2>(j);
      if constexpr (j > 0) {
        const float2 t = tw[j * 16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float q = zr[h][rj];
          zr[h][rj] = fmaf(q, t.x, -zi[h][rj] * t.y);
          zi[h][rj] = fmaf(q, t.y, zi[h][rj] * t.x);
        }
      }
      ha[j * WS] = make_float2(zr[0][rj], zr[1][rj]);
      hmo[j * WS] = make_float2(zi[0][rj], zi[1][rj]);
    });
  }
}

// Last-pass twiddles of one lane k: W_N^{k r} = h[(r >> 2) 64] * w[r & 3] (w[0] = 1, not stored).
struct LTw {
  const float2* h;
  float2 w1, w2, w3;
  template <int R_>
  __device__ __forceinline__ float2 at() const {
    constexpr int a = R_ >> 2, b = R_ & 3;
    const float2 t = h[a * 64];
    if constexpr (b == 0) {
      return t;
    } else {
      const float2 w = b == 1 ? w1 : (b == 2 ? w2 : w3);
      return make_float2(fmaf(t.x, w.x, -t.y * w.y), fmaf(t.x, w.y, t.y * w.x));
    }
  }
};

// Last-pass general set: S_k = {j 128 +- k}, M3 blocks, half pairs hold (Z_j, Z_{j + M3/2}).
template <int M, bool kInv>
__device__ __forceinline__ void p3_last_set(float2* ha, float2* hm, const float2* hmi, float2* hmo, const LTw& tw) {
  constexpr int WS = 4 * 34, LM = ilog2c<M>();  // 128 slots = 4 padded windows
  float zr[M], zi[M];
  if (!kInv) {
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      const float2 a = ha[jj * WS], b = hmi[jj * WS];
      zr[jj] = a.x; zr[jj + M / 2] = a.y;
      zi[jj] = b.x; zi[jj + M / 2] = b.y;
    });
    ct::static_for<1, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 t = tw.template at<rev_bits<LM>(j)>();
      const float q = zr[j];
      zr[j] = fmaf(q, t.x, -zi[j] * t.y);
      zi[j] = fmaf(q, t.y, zi[j] * t.x);
    });
    cfft_dit<M>(zr, zi);
    ct::static_for<0, M / 2>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      ha[q * WS] = make_float2(zr[q], -zi[q + M / 2]);
      hm[(M / 2 - 1 - q) * WS] = make_float2(zr[q + M / 2], zi[q]);
    });
  } else {
    ct::static_for<0, M / 2>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      const float2 a = ha[q * WS], b = hm[(M / 2 - 1 - q) * WS];
      zr[rev_bits<LM>(q)] = a.x;
      zi[rev_bits<LM>(q + M / 2)] = -a.y;
      zr[rev_bits<LM>(q + M / 2)] = b.x;
      zi[rev_bits<LM>(q)] = b.y;
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
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      constexpr int r1 = rev_bits<LM>(jj), r2 = rev_bits<LM>(jj + M / 2);
      ha[jj * WS] = make_float2(zr[r1], zr[r2]);
      hmo[jj * WS] = make_float2(zi[r1], zi[r2]);
    });
  }
}

// Forward last-pass set storing its packed outputs straight to the global row (Plan3::FD):
// da -> slot k of the row, dm -> slot 128 - k; kz: k = 64, whose mirror slot is its own.
template <int M, typename T>
__device__ __forceinline__ void p3_last_set_fwd_direct(const float2* ha, const float2* hmi, const LTw& tw, T* da,
                                                       T* dm, bool kz, int n) {
  constexpr int WS = 4 * 34, LM = ilog2c<M>();
  float zr[M], zi[M];
  ct::static_for<0, M / 2>([&](auto J) {
    constexpr int jj = decltype(J)::value;
    const float2 a = ha[jj * WS], b = hmi[jj * WS];
    zr[jj] = a.x; zr[jj + M / 2] = a.y;
    zi[jj] = b.x; zi[jj + M / 2] = b.y;
  });
  ct::static_for<1, M>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const float2 t = tw.template at<rev_bits<LM>(j)>();
    const float q = zr[j];
    zr[j] = fmaf(q, t.x, -zi[j] * t.y);
    zi[j] = fmaf(q, t.y, zi[j] * t.x);
  });
  cfft_dit<M>(zr, zi);
  ct::static_for<0, M / 2>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    gio<T>::st1(da + q * 128, zr[q]);
    gio<T>::st1(da + q * 128 + n / 2, -zi[q + M / 2]);
    if (!kz) {
      gio<T>::st1(dm + (M / 2 - 1 - q) * 128, zr[q + M / 2]);
      gio<T>::st1(dm + (M / 2 - 1 - q) * 128 + n / 2, zi[q]);
    }
  });
}

// Forward last-pass DC set (slots j 128, j 128 + n/2) from H, stored straight to the global row.
template <int M, typename T>
__device__ __forceinline__ void p3_dc_fwd_direct(const float2* hd, T* d0, int n) {
  constexpr int WS = 4 * 34;
  float d[M];
  ct::static_for<0, M / 2>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const float2 a = hd[j * WS];
    d[j] = a.x;
    d[j + M / 2] = a.y;
  });
  rfft_fwd_reg<M>(d);
  ct::static_for<0, M / 2>([&](auto J) {
    constexpr int j = decltype(J)::value;
    gio<T>::st1(d0 + j * 128, d[j]);
    gio<T>::st1(d0 + j * 128 + n / 2, d[j + M / 2]);
  });
}

// Inverse last-pass set read straight from the staged tile (natural order, element type T): the
// values p3_last_set<M, true> would read from H after the load phase copied them there.
template <int M, typename T, typename LD = sio1<T>>
__device__ __forceinline__ void p3_last_set_inv_st(const T* sa, const T* sm, float2* ha, float2* hmo, const LTw& tw,
                                                   int n, uint32_t k65536) {
  constexpr int WS = 4 * 34, LM = ilog2c<M>();
  float zr[M], zi[M];
  ct::static_for<0, M / 2>([&](auto Q) {
    constexpr int q = decltype(Q)::value;
    zr[rev_bits<LM>(q)] = LD::ld(sa + q * 128, k65536);
    zi[rev_bits<LM>(q + M / 2)] = -LD::ld(sa + q * 128 + n / 2, k65536);
    zr[rev_bits<LM>(q + M / 2)] = LD::ld(sm + (M / 2 - 1 - q) * 128, k65536);
    zi[rev_bits<LM>(q)] = LD::ld(sm + (M / 2 - 1 - q) * 128 + n / 2, k65536);
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
  ct::static_for<0, M / 2>([&](auto J) {
    constexpr int jj = decltype(J)::value;
    constexpr int r1 = rev_bits<LM>(jj), r2 = rev_bits<LM>(jj + M / 2);
    ha[jj * WS] = make_float2(zr[r1], zr[r2]);
    hmo[jj * WS] = make_float2(zi[r1], zi[r2]);
  });
}

// Inverse last-pass DC set from the staged tile: slots j 128 and j 128 + n/2 -> H half pairs.
template <int M, typename T, typename LD = sio1<T>>
__device__ __forceinline__ void p3_dc_inv_st(const T* s, float2* hd, int n, uint32_t k65536) {
  constexpr int WS = 4 * 34;
  float d[M];
  ct::static_for<0, M / 2>([&](auto J) {
    constexpr int j = decltype(J)::value;
    d[j] = LD::ld(s + j * 128, k65536);
    d[j + M / 2] = LD::ld(s + j * 128 + n / 2, k65536);
  });
  rfft_inv_reg<M>(d);
  const float sc = 1.0f / (float)n;
  ct::static_for<0, M / 2>([&](auto J) {
    constexpr int j = decltype(J)::value;
    hd[j * WS] = make_float2(d[j] * sc, d[j + M / 2] * sc);
  });
}

// DC set of a pass: M reals-pairs at stride WS (float2 lanes), real M-point FFT (unscaled inverse).
template <int M, int WS, bool kInv, typename V>
__device__ __forceinline__ void p3_dc_set(float2* hd, float scale) {
  V d[M];
  ct::static_for<0, (sizeof(V) == 8 ? M : M / 2)>([&](auto J) {
    constexpr int j = decltype(J)::value;
    if constexpr (sizeof(V) == 8) {
      d[j] = *reinterpret_cast<V*>(hd + j * WS);
    } else {  // scalar lanes: (D_j, D_{j + M/2}) in one half pair
      const float2 a = hd[j * WS];
      reinterpret_cast<float*>(d)[j] = a.x;
      reinterpret_cast<float*>(d)[j + M / 2] = a.y;
    }
  });
  if (!kInv)
    rfft_fwd_reg<M>(d);
  else
    rfft_inv_reg<M>(d);
  ct::static_for<0, (sizeof(V) == 8 ? M : M / 2)>([&](auto J) {
    constexpr int j = decltype(J)::value;
    if constexpr (sizeof(V) == 8) {
      const float2 v = *reinterpret_cast<float2*>(&d[j]);
      hd[j * WS] = make_float2(v.x * scale, v.y * scale);
    } else {
      hd[j * WS] = make_float2(reinterpret_cast<float*>(d)[j] * scale, reinterpret_cast<float*>(d)[j + M / 2] * scale);
    }
  });
}

template <typename P, bool kInv>
__global__ void __launch_bounds__(P::NT) rdfft3_kernel(typename P::elem* __restrict__ x, int64_t batch) {
  using T = typename P::elem;
  using L = P3Smem<P>;
  constexpr int VT = P::VT, N = P::N, NT = P::NT, R = P::R, S = P::S, WS = P::WSTR;
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float2* H = reinterpret_cast<float2*>(base + L::H_OFF);
  float2* TWm = reinterpret_cast<float2*>(base + L::TWM_OFF);
  float2* TWl = reinterpret_cast<float2*>(base + L::TWL_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  const int tid = threadIdx.x;
  // tables: TWm[j 16 + k-1] = W_128^{k rev2(j)}; TWl (see Plan3::TWL); inverse: conj (and 1/N on TWl)
  for (int e = tid; e < P::TWM; e += NT) {
    const int j = e / 16, k = 1 + e % 16;
    float s, c;
    sincospif(2.0f * (float)(k * rev_bits<2>(j)) / 128.0f, &s, &c);
    TWm[e] = kInv ? make_float2(c, s) : make_float2(c, -s);
  }
  for (int e = tid; e < P::TWL; e += NT) {  // TWl[a 64 + k-1] = W_N^{4 k a} (inverse: conj / N)
    const int a = e / 64, k = 1 + e % 64;
    float s, c;
    sincospif(2.0f * (float)(4 * k * a) / (float)N, &s, &c);
    TWl[e] = kInv ? make_float2(c * (1.0f / N), s * (1.0f / N)) : make_float2(c, -s);
  }
  for (int e = tid; e < P::NWIN * VT; e += NT) {  // window pads (zero imaginary inputs)
    float2* pad = H + P::row(e / P::NWIN) + (e % P::NWIN) * WS + R;
    pad[0] = make_float2(0.f, 0.f);
    pad[1] = make_float2(0.f, 0.f);
  }
  if (tid == 0) {
    for (int q = 0; q < (P::NSTG > 0 ? P::NSTG : 1); ++q) mbar_init(bar + q, 1);
    fence_mbar_init();
  }
  // ---- roles
  const int v1 = tid / P::P1, w1 = tid % P::P1;
  const int c1 = rev_bits<P::LS - 1>(w1);
  float2* h1 = H + P::row(v1) + w1 * WS;
  const int s1 = v1 * N + 2 * c1;
  // middle general: item it = tid + NT r -> vector vm0 + dv(r), window wm + dw(r), k km (tid-part fixed)
  const int mrem = tid % P::MIPV;
  const int vm0 = NT >= P::MIPV ? tid / P::MIPV : 0;
  const int wm = mrem / P::KM, km = 1 + mrem % P::KM;
  float2* mha = H + P::row(vm0) + 4 * wm * WS + km;
  float2* mhm = H + P::row(vm0) + 4 * wm * WS + (R - km);
  float2* mhz = (km == R / 2) ? (H + P::row(vm0) + 4 * wm * WS + R) : mhm;  // pad: zero input / sink
  const float2* mtw = TWm + (km - 1);
  constexpr int MITEMS = VT * P::MIPV / NT;
  // middle DC items: (vector, window), VT * WPV of them, on the last threads
  constexpr int NDCM = VT * P::WPV;
  const int dcm = tid - (NT - NDCM);
  float2* mhd = H + P::row(dcm < 0 ? 0 : dcm / P::WPV) + 4 * ((dcm < 0 ? 0 : dcm) % P::WPV) * WS;
  // last general: item it = tid + NT r -> vector vl0 + r LSTEP, k kl
  const int vl0 = tid / P::KL, kl = 1 + tid % P::KL;
  const int qa = kl, qm = P::W2 - kl;
  float2* lha = H + P::row(vl0) + P::pos(qa);
  float2* lhm = H + P::row(vl0) + P::pos(qm);
  float2* lhz = (kl == P::KL) ? (H + P::row(vl0) + P::pos(qa) + (R - (qa % R))) : lhm;
  LTw ltw;
  ltw.h = TWl + (kl - 1);
  {
    float s1, c1, s2, c2, s3, c3;
    sincospif(2.0f * (float)kl / (float)N, &s1, &c1);
    sincospif(4.0f * (float)kl / (float)N, &s2, &c2);
    sincospif(6.0f * (float)kl / (float)N, &s3, &c3);
    const float sg = kInv ? 1.0f : -1.0f;
    ltw.w1 = make_float2(c1, sg * s1);
    ltw.w2 = make_float2(c2, sg * s2);
    ltw.w3 = make_float2(c3, sg * s3);
  }
  constexpr int LSTEP = NT / P::KL;
  constexpr int LITEMS = VT * P::KL / NT;
  const int dcl = tid - (NT - VT);  // last DC: one lane per vector on the last threads
  float2* lhd = H + P::row(dcl < 0 ? 0 : dcl);
  // chunks
  float2* hq = H + (2 * tid / R) * WS + (2 * tid) % R;
  const uint32_t k65536 = kTwo16;
  const int64_t ntiles = (batch + VT - 1) / VT;
  auto tile_bytes = [&](int64_t t) {
    const int64_t nv = batch - t * VT < VT ? batch - t * VT : VT;
    return (uint32_t)(nv * N * (int)sizeof(T));
  };
  __syncthreads();
  constexpr int NS = P::NSTG;
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) {
      const int64_t t = blockIdx.x + (int64_t)q * gridDim.x;
      if (t < ntiles) stage_issue(x + t * VT * (int64_t)N, tile_bytes(t), base + q * P::STAGE, bar + q);
    }
  }
  auto middle = [&](int nv) {
    ct::static_for<0, MITEMS>([&](auto RR) {
      constexpr int r = decltype(RR)::value;
      // NT >= MIPV: item step = NT / MIPV vectors;  NT < MIPV: MIPV / NT steps per vector, each
      // NT / 16 windows further along the same row
      constexpr int dv = NT >= P::MIPV ? r * (NT / P::MIPV) : r / (P::MIPV / NT);
      constexpr int dwin = NT >= P::MIPV ? 0 : (r % (P::MIPV / NT)) * (NT / P::KM);
      constexpr int off = dv * P::ROWA + 2 * dv + dwin * 4 * WS;  // row(vm0 + dv) - row(vm0), v < 8
      if (vm0 + dv < nv) p3_mid_set<kInv>(mha + off, mhm + off, mhz + off, mhz + off, mtw);
    });
    if (dcm >= 0 && dcm / P::WPV < nv) p3_dc_set<4, WS, kInv, float2>(mhd, 1.0f);
  };
  auto last = [&](int nv) {
    ct::static_for<0, LITEMS>([&](auto RR) {
      constexpr int r = decltype(RR)::value;
      constexpr int dv = r * LSTEP;
      constexpr int off = dv * P::ROWA + 2 * dv;
      if (vl0 + dv < nv) p3_last_set<P::M3, kInv>(lha + off, lhm + off, lhz + off, lhz + off, ltw);
    });
    if (dcl >= 0 && dcl < nv) p3_dc_set<P::M3, 4 * WS, kInv, float>(lhd, kInv ? 1.0f / N : 1.0f);
  };
  // the inverse's first pass, reading the staged tile (NSTG > 0) or the global tile (NSTG = 0)
  using LD = std::conditional_t<(P::NSTG > 0), sio1<T>, gio1<T>>;
  auto last_inv_st = [&](const T* st, int nv) {
    ct::static_for<0, LITEMS>([&](auto RR) {
      constexpr int r = decltype(RR)::value;
      constexpr int dv = r * LSTEP;
      constexpr int off = dv * P::ROWA + 2 * dv;
      const T* sv = st + (vl0 + dv) * N;
      if (vl0 + dv < nv) p3_last_set_inv_st<P::M3, T, LD>(sv + qa, sv + qm, lha + off, lhz + off, ltw, N, k65536);
    });
    if (dcl >= 0 && dcl < nv) p3_dc_inv_st<P::M3, T, LD>(st + dcl * N, lhd, N, k65536);
  };
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int nv = (int)(batch - tile * VT < VT ? batch - tile * VT : VT);
    T* xt = x + tile * VT * (int64_t)N;
    const int sb = NS > 0 ? it % NS : 0;
    const T* st = NS > 0 ? reinterpret_cast<const T*>(base + sb * P::STAGE) : xt;
    const int64_t nxt = tile + NS * (int64_t)gridDim.x;
    if constexpr (NS > 0) mbar_wait(bar + sb, (it / NS) & 1);
    if (!kInv) {
      if (v1 < nv) {  // pass 1 (plan2's)
        float2 b[R];
        const T* src = st + s1;
        ct::static_for<0, R>([&](auto I) {
          constexpr int i = decltype(I)::value;
          if constexpr (NS > 0)
            b[rev_bits<P::LR>(i)] = sio<T>::ld2(src + S * i, k65536);
          else
            b[rev_bits<P::LR>(i)] = gio<T>::ld2(src + S * i, k65536);
        });
        rfft_fwd_reg<R>(b);
        ct::static_for<0, R / 2>([&](auto I) {
          constexpr int i = 2 * decltype(I)::value;
          *reinterpret_cast<float4*>(h1 + i) = make_float4(b[i].x, b[i].y, b[i + 1].x, b[i + 1].y);
        });
      }
      __syncthreads();
      if (NS > 0 && tid == 0 && nxt < ntiles) stage_issue(x + nxt * VT * (int64_t)N, tile_bytes(nxt), base + sb * P::STAGE, bar + sb);
      middle(nv);
      __syncthreads();
      if constexpr (P::FD) {
        ct::static_for<0, LITEMS>([&](auto RR) {
          constexpr int r = decltype(RR)::value;
          constexpr int dv = r * LSTEP;
          constexpr int off = dv * P::ROWA + 2 * dv;
          T* xv = xt + (vl0 + dv) * N;
          if (vl0 + dv < nv) p3_last_set_fwd_direct<P::M3, T>(lha + off, lhz + off, ltw, xv + qa, xv + qm, kl == P::KL, N);
        });
        if (dcl >= 0 && dcl < nv) p3_dc_fwd_direct<P::M3, T>(lhd, xt + dcl * N, N);
      } else {
      last(nv);
      __syncthreads();
      ct::static_for<0, VT * P::CHV / NT>([&](auto RR) {  // store
        constexpr int r = decltype(RR)::value;
        constexpr int v = r / (P::CHV / NT), toff = NT * (r % (P::CHV / NT));
        if (v < nv) {
          const float4 f = *reinterpret_cast<const float4*>(hq + P::row(v) + (2 * toff / R) * WS);
          T* d = xt + v * N + 2 * (tid + toff);
          gio<T>::st2(d, make_float2(f.x, f.z));
          gio<T>::st2(d + N / 2, make_float2(f.y, f.w));
        }
      });
      }
    } else {
      last_inv_st(st, nv);  // reads the staged tile directly (no staged -> H copy)
      __syncthreads();
      if (NS > 0 && tid == 0 && nxt < ntiles) stage_issue(x + nxt * VT * (int64_t)N, tile_bytes(nxt), base + sb * P::STAGE, bar + sb);
      middle(nv);
      __syncthreads();
      if (v1 < nv) {  // inverse pass 1
        float2 b[R];
        ct::static_for<0, R / 2>([&](auto I) {
          constexpr int i = 2 * decltype(I)::value;
          const float4 f = *reinterpret_cast<const float4*>(h1 + i);
          b[i] = make_float2(f.x, f.y);
          b[i + 1] = make_float2(f.z, f.w);
        });
        rfft_inv_reg<R>(b);
        T* dst = xt + s1;
        ct::static_for<0, R>([&](auto I) {
          constexpr int i = decltype(I)::value;
          gio<T>::st2(dst + S * i, b[rev_bits<P::LR>(i)]);
        });
      }
    }
    __syncthreads();
  }
}

template <typename P, bool kInv>
bool launch_plan3_dir(typename P::elem* x, int64_t batch, int sms, cudaStream_t st) {
  using L = P3Smem<P>;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  auto k = rdfft3_kernel<P, kInv>;
  static int per_sm_dev[kMaxDevices] = {};
  int& per_sm = per_sm_dev[device_index()];
  if (!per_sm) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, P::NT, L::BYTES);
    if (per_sm < 1) per_sm = 1;
    if (verbose())
      std::fprintf(stderr, "[rdfft] plan3 n=%d VT=%d NSTG=%d inv=%d: %zu B smem, %d threads, %d CTAs/SM\n", P::N,
                   P::VT, P::NSTG, (int)kInv, (size_t)L::BYTES, P::NT, per_sm);
  }
  const int64_t tiles = (batch + P::VT - 1) / P::VT;
  const int grid = (int)(tiles < (int64_t)per_sm * sms ? tiles : (int64_t)per_sm * sms);
  k<<<grid, P::NT, L::BYTES, st>>>(x, batch);
  return true;
}
// forward plan PF, inverse plan PI
template <typename PF, typename PI>
bool launch_plan3(typename PF::elem* x, int64_t batch, bool inverse, int sms, cudaStream_t st) {
  return inverse ? launch_plan3_dir<PI, true>(x, batch, sms, st) : launch_plan3_dir<PF, false>(x, batch, sms, st);
}

#ifndef RDFFT_FWD_NSTG
#define RDFFT_FWD_NSTG 1  // forward staging depth for n = 512 / 1024 (0 = pass 1 straight from HBM)
#endif
// Returns true when a specialised kernel was launched for (n, T).
// bf16 forward, n = 256..1024: the output-staged kernel (rdfft2fo_kernel, plan2.cuh), measured against
// the H -> HBM store phase of rdfft2_kernel (2^20 vectors, fraction of HBM; gpurun_out r02_h):
// n = 1024 0.721 -> 0.799 (6 vectors per CTA, 4 CTAs/SM; 8 vectors at 3 CTAs/SM: 0.783), 512
// 0.683 -> 0.710, 256 0.664 -> 0.702 (12 vectors per CTA); pass 1 straight from HBM instead of the
// staging buffer measured 0.58-0.62 at every n.
// bf16 inverse, n = 256..1024: the staged-read kernel (plan2o.cuh; measured 64 -> 70-76 % of HBM at
// 512/1024; an output tile for its pass 1 measured equal or slower: 0.688 -> 0.684, 0.733 -> 0.717,
// 0.772 -> 0.703, r02_i).  (bf16 n = 128 runs the transposing one-vector-per-thread kernel, small.cuh.)
template <typename T, int N, int R, int VT>
bool launch_p2(T* x, int64_t batch, bool inverse, int sms, cudaStream_t st) {
  if constexpr (sizeof(T) == 2 && N >= 256) {
    if (!inverse) {
      constexpr int VTF = R == 32 ? (N == 1024 ? 6 : VT) : 12;
      return launch_plan2fo<Plan2<T, N, R, VTF, 1>>(x, batch, sms, st);
    }
    // n = 256 / 512: 2-deep TMA ring (0.71 -> 0.74 of HBM at 512; at 1024 it costs a CTA per SM:
    // 0.77 -> 0.75; n = 256 0.60 -> 0.68 with the per-width staging skew)
    return launch_plan2o_inv<Plan2o<N, R, VT, ((N == 512 || N == 256) ? 2 : 1)>>(x, batch, sms, st);
  } else {
    return launch_plan2<Plan2<T, N, R, VT, (N >= 512 ? RDFFT_FWD_NSTG : 2)>, Plan2<T, N, R, VT, (N >= 512 ? 1 : 2)>>(
        x, batch, inverse, sms, st);
  }
}

template <typename T>
bool launch_rdfft_fast(T* x, int64_t batch, int n, int logn, bool inverse, int sms, cudaStream_t st) {
  (void)logn;
  switch (n) {
    case 2: return launch_small<T, 2>(x, batch, inverse, sms, st);
    case 4: return launch_small<T, 4>(x, batch, inverse, sms, st);
    case 8: return launch_small<T, 8>(x, batch, inverse, sms, st);
    case 16: return launch_small<T, 16>(x, batch, inverse, sms, st);
    case 32: return launch_small<T, 32>(x, batch, inverse, sms, st);
    // n = 64 (both dtypes) and bf16 n = 128: one vector per thread through the per-warp shared-memory
    // transpose (small.cuh).  Against the two-pass plan (2^20 vectors, fraction of HBM, gpurun_out
    // r02_y): fp32 n = 64 0.80 / 0.60 -> 0.95 / 0.95, bf16 n = 128 0.64 / 0.60 -> 0.82 / 0.86
    case 64: return launch_small<T, 64>(x, batch, inverse, sms, st);
    case 128:
      if constexpr (sizeof(T) == 2) return launch_small<T, 128>(x, batch, inverse, sms, st);
      else return launch_p2<T, 128, 16, 32>(x, batch, inverse, sms, st);
    case 256: return launch_p2<T, 256, 16, (sizeof(T) == 4 ? 32 : 16)>(x, batch, inverse, sms, st);
    case 512: return launch_p2<T, 512, 32, 8>(x, batch, inverse, sms, st);
    case 1024: return launch_p2<T, 1024, 32, 8>(x, batch, inverse, sms, st);
    // bf16 n = 2048 forward: the last pass writes an output tile stored by TMA (0.592 -> 0.622 of HBM,
    // 3 CTAs/SM; the inverse through an output tile measured 0.627 -> 0.597 and n = 4096 0.533 / 0.54 ->
    // 0.53 / 0.52, r02_j): both keep the direct stores
    // n = 2048: the two-pass R = 64 plan (plan2s.cuh) for the bf16 forward (with the output tile, 3
    // vectors per CTA) and the fp32 inverse; plan3 elsewhere (fraction of HBM, 2^20 vectors, r02_o:
    // bf16 fwd plan3 0.622 -> plan2s 0.706, fp32 inv 0.916 -> 0.970; bf16 inv 0.631 -> 0.583-0.598 and
    // fp32 fwd 0.919 -> 0.889-0.924 stay on plan3)
    case 2048:
      if constexpr (sizeof(T) == 2) {
        if (!inverse) return launch_plan2s_dir<Plan2s<T, 2048, 3, true>, false>(x, batch, sms, st);
        return launch_plan3_dir<Plan3<T, 2048, 4, 1, true>, true>(x, batch, sms, st);
      } else {
        if (inverse) return launch_plan2s_dir<Plan2s<T, 2048, 4>, true>(x, batch, sms, st);
        return launch_plan3_dir<Plan3<T, 2048, 4, 1, true>, false>(x, batch, sms, st);
      }
    case 4096: return launch_plan3<Plan3<T, 4096, 2, 1, true>, Plan3<T, 4096, 2, 1, true>>(x, batch, inverse, sms, st);
    case 8192: return launch_planl<PlanL<T, 8192>>(x, batch, inverse, sms, st);
    case 16384: return launch_planl<PlanL<T, 16384>>(x, batch, inverse, sms, st);
    case 32768: return launch_planl<PlanL<T, 32768>>(x, batch, inverse, sms, st);
    case 65536: return launch_planl_pair<PlanL<T, 32768>>(x, batch, inverse, sms, st);
    default: return false;
  }
}

}  // namespace rdfft
