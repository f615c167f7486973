// regfft.cuh — in-register sub-transforms with compile-time twiddles.
//
//  * rfft_fwd_reg<R>  : the paper's forward stages (Prop. 1) on R
//                       reals already in bit-reversed order -> packed R-point
//                       spectrum.  Operates on float2 "lanes": two
//                       independent sequences transformed together.
//  * rfft_inv_reg<R>  : the reversed graph (Eq. 7), UNSCALED: every
//                       stage is 2x the paper's stage (the 1/2 is dropped on the
//                       k = 0 pair and the groups, and the k = m/2 slots are
//                       doubled instead), so the composition is R x the true
//                       inverse; callers fold the 1/n once (reading C4: per-stage
//                       halving and one final 1/n are bit-identical in binary FP).
//  * cfft_dit<M> / cfft_dif_inv<M> : complex radix-2 FFTs used for the
//                       register-blocked last pass (see rdfft_kernels.cuh).
#pragma once

#include "ct.cuh"

namespace rdfft {

__device__ __forceinline__ float2 operator+(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 operator-(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 operator-(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 operator*(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 fma2s(float2 a, float s, float2 c) {
  return make_float2(fmaf(a.x, s, c.x), fmaf(a.y, s, c.y));
}
__device__ __forceinline__ float fma2s(float a, float s, float c) { return fmaf(a, s, c); }

// ------------------------------------------------------------------ real FFT
// b: R lanes in bit-reversed order -> packed spectrum.  Lane type V is float2.
template <int R, typename V>
__device__ __forceinline__ void rfft_fwd_reg(V (&b)[R]) {
  ct::static_for<0, 31>([&](auto LM) {
    constexpr int m = 1 << decltype(LM)::value;
    if constexpr (m < R) {
      ct::static_for<0, R / (2 * m)>([&](auto BB) {
        constexpr int be = decltype(BB)::value * 2 * m;
        {  // k = 0: both bins real
          const V a = b[be], c = b[be + m];
          b[be] = a + c;
          b[be + m] = a - c;
        }
        if constexpr (m >= 2) b[be + 3 * m / 2] = -b[be + 3 * m / 2];  // k = m/2
        ct::static_for<1, m / 2>([&](auto KK) {
          constexpr int k = decltype(KK)::value;
          const V Ar = b[be + k], Ai = b[be + m - k], Br = b[be + m + k], Bi = b[be + 2 * m - k];
          // u = W B with W = W_{2m}^k written as g (1 + i tau) (k < m/4) or g (tau + i)
          // (k > m/4): B' = B (1 + i tau) costs 2 FFMA and the outputs A +- g B' 4 FFMA.
          V Bpr, Bpi;
          float g;
          if constexpr (4 * k == m) {  // W = (1 - i)/sqrt2
            Bpr = Br + Bi;
            Bpi = Bi - Br;
            g = ct::W<k, 2 * m>::re;
          } else if constexpr (4 * k < m) {
            constexpr float tau = ct::Wt<k, 2 * m>::tan;
            Bpr = fma2s(Bi, -tau, Br);
            Bpi = fma2s(Br, tau, Bi);
            g = ct::W<k, 2 * m>::re;
          } else {
            constexpr float tau = ct::Wt<k, 2 * m>::cot;
            Bpr = fma2s(Br, tau, -Bi);
            Bpi = fma2s(Bi, tau, Br);
            g = ct::W<k, 2 * m>::im;
          }
          b[be + k] = fma2s(Bpr, g, Ar);
          b[be + 2 * m - k] = fma2s(Bpi, g, Ai);
          b[be + m - k] = fma2s(Bpr, -g, Ar);
          b[be + m + k] = fma2s(Bpi, g, -Ai);
        });
      });
    }
  });
}

// Packed spectrum -> R x (bit-reversed real sequence).  Unscaled (see header).
// The doubling of the k = m/2 slots is folded into the next stage: those slots are exactly the
// k = 0 partners (b[be + m]) of the following stage, which then combines a +- 2c with one FFMA.
template <int R, typename V>
__device__ __forceinline__ void rfft_inv_reg(V (&b)[R]) {
  ct::static_for<0, 31>([&](auto LI) {
    constexpr int lm = 30 - decltype(LI)::value;  // descending stage order
    constexpr int m = 1 << lm;
    if constexpr (m < R) {
      constexpr bool first = (2 * m == R);  // inputs all at the same scale
      ct::static_for<0, R / (2 * m)>([&](auto BB) {
        constexpr int be = decltype(BB)::value * 2 * m;
        {
          const V a = b[be], c = b[be + m];
          if constexpr (first) {
            b[be] = a + c;
            b[be + m] = a - c;
          } else {  // c is an undoubled k = m/2 slot of the previous stage
            b[be] = fma2s(c, 2.0f, a);
            b[be + m] = fma2s(c, -2.0f, a);
          }
        }
        if constexpr (m >= 2) b[be + 3 * m / 2] = -b[be + 3 * m / 2];  // k = m/2: sign only
        ct::static_for<1, m / 2>([&](auto KK) {
          constexpr int k = decltype(KK)::value;
          // B = (Yk - Y_{m+k}) conj(W): conj(W) = (wr, -wi)
          constexpr float wr = ct::W<k, 2 * m>::re, wi = ct::W<k, 2 * m>::im;
          const V Ykr = b[be + k], Yki = b[be + 2 * m - k];
          const V Ymr = b[be + m - k], Ymi = -b[be + m + k];  // Y_{m+k} = conj(Y_{m-k})
          const V dr = Ykr - Ymr, di = Yki - Ymi;
          b[be + k] = Ykr + Ymr;
          b[be + m - k] = Yki + Ymi;
          if constexpr (4 * k == m) {  // conj(W) = (1 + i)/sqrt2
            b[be + m + k] = (dr - di) * wr;
            b[be + 2 * m - k] = (dr + di) * wr;
          } else {
            b[be + m + k] = fma2s(dr, wr, di * wi);
            b[be + 2 * m - k] = fma2s(di, wr, dr * (-wi));
          }
        });
      });
    }
  });
}

// ---------------------------------------------------------------- complex FFT
// Multiply (xr, xi) by the compile-time W_{2h}^l (or its conjugate) in place.
template <int L, int H2, bool kConj>
__device__ __forceinline__ void cmul_ct(float& xr, float& xi) {
  constexpr int l = L % H2;
  if constexpr (l == 0) {
    return;
  } else if constexpr (4 * l == H2) {  // W = -i (conj: +i)
    const float r = xr;
    if constexpr (kConj) {
      xr = -xi;
      xi = r;
    } else {
      xr = xi;
      xi = -r;
    }
  } else {
    constexpr float wr = ct::W<l, H2>::re;
    constexpr float wi = kConj ? -ct::W<l, H2>::im : ct::W<l, H2>::im;
    if constexpr (8 * l == H2 || 8 * l == 3 * H2 || 8 * l == 5 * H2 || 8 * l == 7 * H2) {
      // |wr| == |wi| == sqrt(1/2): (xr wr - xi wi, xr wi + xi wr) with 2 mul + 2 add
      constexpr float s = wr > 0 ? wr : -wr;
      constexpr bool pr = wr > 0, pi = wi > 0;
      const float a = pr ? xr : -xr;   // xr * sign(wr)
      const float bq = pi ? xi : -xi;  // xi * sign(wi)
      const float c = pi ? xr : -xr;   // xr * sign(wi)
      const float d = pr ? xi : -xi;   // xi * sign(wr)
      xr = (a - bq) * s;
      xi = (c + d) * s;
    } else {
      const float r = xr;
      xr = fmaf(r, wr, -xi * wi);
      xi = fmaf(r, wi, xi * wr);
    }
  }
}

// Radix-2 butterfly (a, b) -> (a + W b, a - W b) with compile-time W = W_{H2}^L (conj if kConj).
// Non-trivial W = g (1 + i tau): b' = b (1 + i tau) in 2 FFMA, then a +- g b' in 4 FFMA.
template <int L, int H2, bool kConj>
__device__ __forceinline__ void bfly_ct(float& ar, float& ai, float& br, float& bi) {
  constexpr int l = L % H2;
  if constexpr (l == 0 || 4 * l == H2) {
    float tr = br, ti = bi;
    cmul_ct<l, H2, kConj>(tr, ti);
    br = ar - tr;
    bi = ai - ti;
    ar = ar + tr;
    ai = ai + ti;
  } else {
    constexpr float wr = ct::W<l, H2>::re;
    constexpr float wi = kConj ? -ct::W<l, H2>::im : ct::W<l, H2>::im;
    constexpr float awr = wr < 0 ? -wr : wr, awi = wi < 0 ? -wi : wi;
    float pr, pi, g;
    if constexpr (8 * l == H2 || 8 * l == 3 * H2 || 8 * l == 5 * H2 || 8 * l == 7 * H2) {
      // W = g (1 + i s) with s = wi / wr = +-1
      constexpr bool sp = (wi > 0) == (wr > 0);
      pr = sp ? br - bi : br + bi;
      pi = sp ? bi + br : bi - br;
      g = wr;
    } else if constexpr (awr >= awi) {
      constexpr float tau = (float)((double)wi / (double)wr);
      pr = fmaf(bi, -tau, br);
      pi = fmaf(br, tau, bi);
      g = wr;
    } else {  // W = g (tau + i), g = wi, tau = wr / wi
      constexpr float tau = (float)((double)wr / (double)wi);
      pr = fmaf(br, tau, -bi);
      pi = fmaf(bi, tau, br);
      g = wi;
    }
    br = fmaf(pr, -g, ar);
    bi = fmaf(pi, -g, ai);
    ar = fmaf(pr, g, ar);
    ai = fmaf(pi, g, ai);
  }
}

// In-place radix-2 DIT complex FFT of size M, bit-reversed input -> natural output.
//   Y[q] = sum_j W_M^{+-q rev(j)} Z[j]     (kConj: positive exponent, unscaled inverse)
template <int M, bool kConj = false>
__device__ __forceinline__ void cfft_dit(float (&re)[M], float (&im)[M]) {
  ct::static_for<0, 31>([&](auto S) {
    constexpr int h = 1 << decltype(S)::value;
    if constexpr (h < M) {
      ct::static_for<0, M / (2 * h)>([&](auto BB) {
        constexpr int be = decltype(BB)::value * 2 * h;
        ct::static_for<0, h>([&](auto LL) {
          constexpr int l = decltype(LL)::value;
          bfly_ct<l, 2 * h, kConj>(re[be + l], im[be + l], re[be + l + h], im[be + l + h]);
        });
      });
    }
  });
}

// In-place radix-2 DIF inverse complex FFT (conjugate twiddles, UNSCALED),
// natural input -> bit-reversed output:  Z[j] = sum_q W_M^{-q rev(j)} Y[q]  (= M x IDFT).
template <int M>
__device__ __forceinline__ void cfft_dif_inv(float (&re)[M], float (&im)[M]) {
  ct::static_for<0, 31>([&](auto S) {
    constexpr int lh = 30 - decltype(S)::value;
    constexpr int h = 1 << lh;
    if constexpr (h < M) {
      ct::static_for<0, M / (2 * h)>([&](auto BB) {
        constexpr int be = decltype(BB)::value * 2 * h;
        ct::static_for<0, h>([&](auto LL) {
          constexpr int l = decltype(LL)::value;
          const float ar = re[be + l], ai = im[be + l];
          float dr = ar - re[be + l + h], di = ai - im[be + l + h];
          re[be + l] = ar + re[be + l + h];
          im[be + l] = ai + im[be + l + h];
          cmul_ct<l, 2 * h, true>(dr, di);
          re[be + l + h] = dr;
          im[be + l + h] = di;
        });
      });
    }
  });
}

template <int B>
__host__ __device__ constexpr int rev_bits(int i) {
  int r = 0;
  for (int k = 0; k < B; ++k) r |= ((i >> k) & 1) << (B - 1 - k);
  return r;
}

template <int N>
__host__ __device__ constexpr int ilog2c() {
  int l = 0;
  while ((1 << l) < N) ++l;
  return l;
}

}  // namespace rdfft
