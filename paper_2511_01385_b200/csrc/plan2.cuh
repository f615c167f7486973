// plan2.cuh — register-blocked in-place rdFFT building blocks for sm_100a.
//
// Plan "2-pass" for n = R * M (R in {16, 32}, 4 <= M <= R):
//
//  pass 1 (stages m = 1 .. R/2 of the paper's schedule):
//    After bit reversal, the first log2 R stages act independently on windows
//    of R consecutive slots; window w holds the packed R-point spectrum of the
//    decimated subsequence x[rev(w) :: n/R] (per-stage invariant, Eq. 6).  A
//    thread loads two adjacent decimated subsequences 2c, 2c+1 (one 4-byte
//    bf16x2 / 8-byte float2 access per element pair), runs the paper's stages
//    in registers with compile-time twiddles, and writes windows rev(2c) and
//    rev(2c) + S/2 (S = n/R).
//
//  last pass (stages m = R .. n/2): by Prop. 1 the four-slot groups of these
//    log2 M stages close over S_k = {j R +- k}, so one
//    thread owns S_k and finishes all remaining stages without exchange.  For
//    1 <= k <= R/2 the stages are regrouped as a twiddle W_n^{k rev(j)} on the
//    M block spectra Z_j(k) followed by an M-point complex DIT FFT (the same
//    radix-2 butterflies, reordered; k = R/2 has zero imaginary input).  The
//    block DCs (slots j R) form a real M-point FFT run by one lane per vector
//    of the last warp.
//
//  Intermediate: fp32 "half pairs" in shared memory, H[q] = (slot q, slot
//  q + n/2), 16-byte pad per R-window (conflict-free 128-bit window writes;
//  the pad also holds the zero imaginary input of lane k = R/2) and a per-row
//  skew.  Every shared access is 8 or 16 bytes, every address is a per-thread
//  base plus a compile-time offset.
//
//  Inverse: the reversed graph (Eq. 7) — last pass first
//  (conjugate twiddles; 1/n folded into its table, reading C4), then the
//  paper's inverse stages in pass 1.
#pragma once

#include "common.cuh"
#include "regfft.cuh"

namespace rdfft {

// 2^16 as a constant-bank operand ptxas cannot fold: u * kTwo16 (= u << 16) then issues as
// IMAD on the full-rate FMA pipe instead of SHF on the half-rate ALU pipe.
__constant__ uint32_t kTwo16 = 65536u;

template <typename T>
struct sio;  // shared-memory pair loads of T (staging buffers)
template <>
struct sio<float> {
  __device__ __forceinline__ static float2 ld2(const float* p, uint32_t) {
    return *reinterpret_cast<const float2*>(p);
  }
};
template <>
struct sio<__nv_bfloat16> {
  __device__ __forceinline__ static float2 ld2(const __nv_bfloat16* p, uint32_t k65536) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    return make_float2(__uint_as_float(u * k65536), __uint_as_float(u & 0xffff0000u));
  }
};

template <typename T>
struct sio1;  // shared-memory single-element loads of T, widened to fp32
template <>
struct sio1<float> {
  __device__ __forceinline__ static float ld(const float* p, uint32_t) { return *p; }
};
template <>
struct sio1<__nv_bfloat16> {
  __device__ __forceinline__ static float ld(const __nv_bfloat16* p, uint32_t k65536) {
    return __uint_as_float((uint32_t)(*reinterpret_cast<const unsigned short*>(p)) * k65536);
  }
};

template <typename T>
struct gio1;  // global single-element loads of T (streaming), widened to fp32 (sio1's interface)
template <>
struct gio1<float> {
  __device__ __forceinline__ static float ld(const float* p, uint32_t) { return __ldcs(p); }
};
template <>
struct gio1<__nv_bfloat16> {
  __device__ __forceinline__ static float ld(const __nv_bfloat16* p, uint32_t k65536) {
    return __uint_as_float((uint32_t)__ldcs(reinterpret_cast<const unsigned short*>(p)) * k65536);
  }
};

template <typename T>
struct gio;  // global pair loads / stores (streaming)
template <>
struct gio<float> {
  __device__ __forceinline__ static float2 ld2(const float* p, uint32_t) {
    return __ldcs(reinterpret_cast<const float2*>(p));
  }
  __device__ __forceinline__ static void st2(float* p, float2 v) { __stcs(reinterpret_cast<float2*>(p), v); }
  __device__ __forceinline__ static void st1(float* p, float v) { __stcs(p, v); }
};
template <>
struct gio<__nv_bfloat16> {
  __device__ __forceinline__ static float2 ld2(const __nv_bfloat16* p, uint32_t k65536) {
    const uint32_t u = __ldcs(reinterpret_cast<const unsigned int*>(p));
    return make_float2(__uint_as_float(u * k65536), __uint_as_float(u & 0xffff0000u));
  }
  __device__ __forceinline__ static void st2(__nv_bfloat16* p, float2 v) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
    __stcs(reinterpret_cast<unsigned int*>(p), *reinterpret_cast<unsigned int*>(&h));
  }
  __device__ __forceinline__ static void st1(__nv_bfloat16* p, float v) {
    __nv_bfloat16 h = __float2bfloat16_rn(v);
    __stcs(reinterpret_cast<unsigned short*>(p), *reinterpret_cast<unsigned short*>(&h));
  }
};

template <typename T, int N_, int R_, int VT_, int NSTG_ = 2, bool FD_ = false>
struct Plan2 {
  using elem = T;
  static constexpr int N = N_, R = R_, VT = VT_;
  // FD: the forward's last pass (and DC lanes) store the packed outputs straight to HBM (one
  // element per lane) instead of H + a chunked store phase.  Off for every plan2 shape: a warp
  // then stores 16 consecutive slots of each of two rows per instruction, measured 0.65 -> 0.33
  // of HBM at bf16 n = 256 and 0.72 -> 0.56 at n = 1024 (plan3, 32 slots of one row, gains).
  static constexpr bool FD = FD_;
  static constexpr int NSTG = NSTG_;  // staging buffers (TMA ring depth) of the stand-alone transforms
  static constexpr int LN = ilog2c<N>();
  static constexpr int LR = ilog2c<R>();
  static constexpr int M = N / R;           // last-pass FFT size (blocks per vector)
  static constexpr int LM = ilog2c<M>();
  static constexpr int S = N / R;           // decimated subsequences per vector
  static constexpr int LS = ilog2c<S>();
  static constexpr int P1 = S / 2;          // pass-1 threads per vector
  static constexpr int LPV = R / 2;         // last-pass lanes per vector: k = 1 .. R/2
  static constexpr int NT = VT * LPV;
  static constexpr int WSTR = R + 2;        // float2 per window (+16 B pad)
  static constexpr int NWIN = S / 2;        // windows per row (first half of the slots)
  static constexpr int ROWA = ((NWIN * WSTR + 14 + 15) / 16) * 16;  // room for the row skew (<= 14, even)
  static constexpr int HF = VT * ROWA + 16;  // float2 in one H region
  static constexpr int TWS = M + 2;         // twiddle row (one per k), padded: 16-byte pair loads, no conflicts
  static constexpr int TWF = LPV * TWS;
  static constexpr int CHV = N / 4;         // 16-byte H chunks per vector
  static constexpr int DC0 = NT - 32;       // first thread of the warp whose lanes run the DC sets
  static constexpr int NTT = NT;            // threads per CTA (Plan2o adds a dedicated DC warp)
  // Staged rows are skewed so that the vectors one pass-1 load instruction touches read disjoint
  // banks: each vector's P1 lanes read P1 x 4 B (bf16 pairs) or P1 x 8 B (float2), so the skew is
  // that width (capped at 64 B: two vectors per 128-byte wavefront or fewer).  n = 1024: 64 B (two
  // vectors per warp, complementary bank halves); bf16 n = 256 / 512: 32 B (four vectors per warp).
  static constexpr int SKEWB_ = (int)(P1 * (sizeof(T) == 2 ? 4 : 8));
  // (at least 16 B: the per-row TMA bulk copies need 16-byte aligned destinations)
  static constexpr int SKEWB = SKEWB_ < 16 ? 16 : (SKEWB_ < 64 ? SKEWB_ : 64);
  static constexpr int SROW = N + SKEWB / (int)sizeof(T);
  static constexpr int STAGE = VT * SROW * (int)sizeof(T);
  static_assert((SROW * (int)sizeof(T)) % 16 == 0, "staged rows must stay 16-byte aligned (TMA bulk copies)");
  static_assert(M <= 2 * R && M >= 4 && (R == 64 || R == 32 || R == 16), "2-pass plan shape");
  static_assert(NT % 32 == 0 && VT * P1 <= NT, "thread mapping");
  static_assert(VT <= 32, "one DC-set lane per vector in the last warp");
  static_assert((VT * CHV) % NT == 0, "chunk mapping");

  // Row skew (float2).  R = 32: a 16-lane shared-memory phase of the last pass holds 8
  // consecutive k of each of the 2 interleaved vectors of a warp (see P2Roles), so the two sit
  // 8 float2 apart.  R = 16 (vector-major lanes): a phase holds 8 k of 2 vectors, likewise.
  // The low bits spread the DC warp (one lane per vector) over the banks.  Skews are even:
  // window bases stay 16-byte aligned.
  static constexpr bool kInterleave = (LPV == 16);
  __host__ __device__ static constexpr int skew(int v) { return (v & 1) * 8 + ((v >> 1) & 3) * 2; }
  __host__ __device__ static constexpr int row(int v) { return v * ROWA + skew(v); }
  // float2 offset of logical half-pair index q (0 <= q < N/2) of vector v
  __host__ __device__ static constexpr int hidx(int v, int q) { return row(v) + (q / R) * WSTR + (q % R); }
};

// Per-thread role pointers of one thread group (lt = thread index inside the group).
template <typename P>
struct P2Roles {
  float2* h1;        // pass 1: window w1 of vector v1
  int v1, s1, s1s;   //   element offset of subsequence 2 c1 in a global / staged tile
  bool act1;
  int v2, k;         // last pass: vector v2, set k
  float2* ha;        //   slots j R + k
  float2* hm;        //   slots (j+1) R - k
  float2* hmz;       //   imaginary input (fwd): the zero pad for k = R/2
  bool kz;           //   k == R/2: the inverse discards the imaginary output (the pad stays zero)
  const float2* twf; //   forward twiddles (column k - 1)
  const float2* twi; //   inverse twiddles
  int dv;            // DC set: lane dv of the last warp (dv < 0: none)
  float2* hd;
  int vq, tq;        // chunk phase: per-thread vector / chunk offsets
  float2* hq;

  __device__ __forceinline__ P2Roles(float2* H, const float2* TWf, const float2* TWi, int lt) {
    constexpr int R = P::R;
    v1 = lt / P::P1;
    const int w1 = lt % P::P1;
    const int c1 = rev_bits<P::LS - 1>(w1);  // rev_LS(2 c1) == w1: lane order = window order
    act1 = lt < P::VT * P::P1;
    h1 = H + P::row(v1) + w1 * P::WSTR;
    s1 = v1 * P::N + 2 * c1;
    s1s = v1 * P::SROW + 2 * c1;
    // Last-pass lanes: the VPW = 32 / LPV vectors of a warp are interleaved (lane = VPW (k-1) + v),
    // so each 16-lane half of a 128-bit twiddle load touches LPV / 2 distinct rows (128 B, one
    // wavefront); with vector-major lanes both halves read the same 16 rows (4 wavefronts).
    // (R = 16 keeps vector-major lanes: measured faster there.)
    constexpr int VPW = P::kInterleave ? 32 / P::LPV : 1;
    v2 = P::kInterleave ? (lt / 32) * VPW + (lt % VPW) : lt / P::LPV;
    k = 1 + (P::kInterleave ? (lt % 32) / VPW : lt % P::LPV);
    ha = H + P::row(v2) + k;
    hm = H + P::row(v2) + (R - k);
    kz = (k == R / 2);
    hmz = kz ? (H + P::row(v2) + R) : hm;
    twf = TWf + (k - 1) * P::TWS;
    twi = TWi + (k - 1) * P::TWS;
    dv = lt - P::DC0;
    hd = H + P::row(dv < 0 ? 0 : dv);
    vq = (P::CHV < P::NT) ? lt / P::CHV : 0;
    tq = (P::CHV < P::NT) ? lt % P::CHV : lt;
    hq = H + P::row(vq) + (2 * tq / R) * P::WSTR + (2 * tq) % R;
  }
};

// Twiddle tables and pads (whole CTA): TWf[(k-1) TWS + j] = W_N^{k rev(j)}, TWi = conj(.)/N.
template <typename P>
__device__ __forceinline__ void p2_tables(float2* TWf, float2* TWi, int tid, int nthreads) {
  for (int e = tid; e < P::TWF; e += nthreads) {
    const int k = 1 + e / P::TWS, j = e % P::TWS;
    if (j >= P::M) continue;
    float s, c;
    sincospif(2.0f * (float)(k * rev_bits<P::LM>(j)) / (float)P::N, &s, &c);
    if (TWf) TWf[e] = make_float2(c, -s);
    if (TWi) TWi[e] = make_float2(c * (1.0f / P::N), s * (1.0f / P::N));
  }
}
template <typename P>
__device__ __forceinline__ void p2_zero_pads(float2* H, int nvec, int tid, int nthreads) {
  for (int e = tid; e < P::NWIN * nvec; e += nthreads) {
    float2* pad = H + P::row(e / P::NWIN) + (e % P::NWIN) * P::WSTR + P::R;
    pad[0] = make_float2(0.f, 0.f);
    pad[1] = make_float2(0.f, 0.f);
  }
}

// ---------------------------------------------------------------- forward pieces
// pass 1 from a staged tile (shared memory, natural order, element type T)
template <typename P, bool kGlobal = false>
__device__ __forceinline__ void p2_pass1_fwd(const P2Roles<P>& r, const typename P::elem* st, int nv,
                                             uint32_t k65536, int hoff = 0) {
  using T = typename P::elem;
  constexpr int R = P::R, S = P::S;
  if (r.act1 && r.v1 < nv) {
    float2 b[R];
    const T* src = st + (kGlobal ? r.s1 : r.s1s);
    ct::static_for<0, R>([&](auto I) {
      constexpr int i = decltype(I)::value;
      if constexpr (kGlobal)
        b[rev_bits<P::LR>(i)] = gio<T>::ld2(src + S * i, k65536);
      else
        b[rev_bits<P::LR>(i)] = sio<T>::ld2(src + S * i, k65536);
    });
    rfft_fwd_reg<R>(b);
    ct::static_for<0, R / 2>([&](auto I) {
      constexpr int i = 2 * decltype(I)::value;
      *reinterpret_cast<float4*>(r.h1 + hoff + i) = make_float4(b[i].x, b[i].y, b[i + 1].x, b[i + 1].y);
    });
  }
}

template <typename P>
__device__ __forceinline__ void p2_last_fwd(const P2Roles<P>& r, int nv, int hoff = 0) {
  constexpr int M = P::M, WSTR = P::WSTR;
  if (r.v2 < nv) {
    float zr[M], zi[M];
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      const float2 a = r.ha[hoff + jj * WSTR];
      const float2 bb = r.hmz[hoff + jj * WSTR];
      zr[jj] = a.x;
      zr[jj + M / 2] = a.y;
      zi[jj] = bb.x;
      zi[jj + M / 2] = bb.y;
    });
    ct::static_for<0, M / 2>([&](auto J2) {
      constexpr int j0 = 2 * decltype(J2)::value;
      const float4 t2 = *reinterpret_cast<const float4*>(r.twf + j0);
      if constexpr (j0 > 0) {
        const float q = zr[j0];
        zr[j0] = fmaf(q, t2.x, -zi[j0] * t2.y);
        zi[j0] = fmaf(q, t2.y, zi[j0] * t2.x);
      }
      const float q1 = zr[j0 + 1];
      zr[j0 + 1] = fmaf(q1, t2.z, -zi[j0 + 1] * t2.w);
      zi[j0 + 1] = fmaf(q1, t2.w, zi[j0 + 1] * t2.z);
    });
    cfft_dit<M>(zr, zi);
    ct::static_for<0, M / 2>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      r.ha[hoff + q * WSTR] = make_float2(zr[q], -zi[q + M / 2]);
      r.hm[hoff + (M / 2 - 1 - q) * WSTR] = make_float2(zr[q + M / 2], zi[q]);
    });
  }
}

template <typename P>
__device__ __forceinline__ void p2_dc_fwd(const P2Roles<P>& r, int nv, int hoff = 0) {
  constexpr int M = P::M, WSTR = P::WSTR;
  if (r.dv >= 0 && r.dv < nv) {  // block DCs j R: packed real M-point DFT (input already bit-reversed)
    float d[M];
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      const float2 a = r.hd[hoff + jj * WSTR];
      d[jj] = a.x;
      d[jj + M / 2] = a.y;
    });
    rfft_fwd_reg<M>(d);
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      r.hd[hoff + jj * WSTR] = make_float2(d[jj], d[jj + M / 2]);
    });
  }
}

// Single-element shared-memory stores of T (output staging tile), narrowed with RNE.
template <typename T>
struct sst1;
template <>
struct sst1<float> {
  __device__ __forceinline__ static void st1(float* p, float v) { *p = v; }
  __device__ __forceinline__ static void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }
};
template <>
struct sst1<__nv_bfloat16> {
  __device__ __forceinline__ static void st1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
  __device__ __forceinline__ static void st2(__nv_bfloat16* p, float2 v) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v.x, v.y);
  }
};

// Forward last pass / DC set writing the packed outputs straight to the global tile (P::FD) or,
// with ST = sst1<T> and RS = the staged row stride, into an output staging tile: the slots
// p2_last_fwd / p2_dc_fwd would write into H, in natural order.
template <typename P, typename ST = gio<typename P::elem>, int RS = P::N>
__device__ __forceinline__ void p2_last_fwd_direct(const P2Roles<P>& r, typename P::elem* dst, int nv) {
  using T = typename P::elem;
  constexpr int M = P::M, WSTR = P::WSTR, R = P::R, N = P::N;
  if (r.v2 < nv) {
    float zr[M], zi[M];
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      const float2 a = r.ha[jj * WSTR];
      const float2 bb = r.hmz[jj * WSTR];
      zr[jj] = a.x;
      zr[jj + M / 2] = a.y;
      zi[jj] = bb.x;
      zi[jj + M / 2] = bb.y;
    });
    ct::static_for<0, M / 2>([&](auto J2) {
      constexpr int j0 = 2 * decltype(J2)::value;
      const float4 t2 = *reinterpret_cast<const float4*>(r.twf + j0);
      if constexpr (j0 > 0) {
        const float q = zr[j0];
        zr[j0] = fmaf(q, t2.x, -zi[j0] * t2.y);
        zi[j0] = fmaf(q, t2.y, zi[j0] * t2.x);
      }
      const float q1 = zr[j0 + 1];
      zr[j0 + 1] = fmaf(q1, t2.z, -zi[j0 + 1] * t2.w);
      zi[j0 + 1] = fmaf(q1, t2.w, zi[j0 + 1] * t2.z);
    });
    cfft_dit<M>(zr, zi);
    T* da = dst + r.v2 * RS + r.k;        // slots q R + k (and + N/2)
    T* dm = dst + r.v2 * RS + (R - r.k);  // slots q R + R - k
    ct::static_for<0, M / 2>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      ST::st1(da + q * R, zr[q]);
      ST::st1(da + q * R + N / 2, -zi[q + M / 2]);
      if (!r.kz) {  // k = R/2: the mirror slot is the same slot (written from the ascending side)
        ST::st1(dm + (M / 2 - 1 - q) * R, zr[q + M / 2]);
        ST::st1(dm + (M / 2 - 1 - q) * R + N / 2, zi[q]);
      }
    });
  }
}

template <typename P, typename ST = gio<typename P::elem>, int RS = P::N>
__device__ __forceinline__ void p2_dc_fwd_direct(const P2Roles<P>& r, typename P::elem* dst, int nv) {
  using T = typename P::elem;
  constexpr int M = P::M, WSTR = P::WSTR, R = P::R, N = P::N;
  if (r.dv >= 0 && r.dv < nv) {
    float d[M];
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      const float2 a = r.hd[jj * WSTR];
      d[jj] = a.x;
      d[jj + M / 2] = a.y;
    });
    rfft_fwd_reg<M>(d);
    T* dd = dst + r.dv * RS;
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      ST::st1(dd + jj * R, d[jj]);
      ST::st1(dd + jj * R + N / 2, d[jj + M / 2]);
    });
  }
}

// Visit this thread's 16-byte H chunks: f(vv, t, h) with vv the vector, t the chunk index
// (slots 2t, 2t+1 and +N/2) and h the chunk's float2 address.  Chunk (vv, t) lives at
// row(vv) + (2t / R) WSTR + 2t % R; the per-thread base hq covers (vq, tq).
template <typename P, typename F>
__device__ __forceinline__ void p2_chunks(const P2Roles<P>& r, F&& f) {
  constexpr int CPT = P::VT * P::CHV / P::NT;
  ct::static_for<0, CPT>([&](auto RR) {
    constexpr int rr = decltype(RR)::value;
    if constexpr (P::CHV >= P::NT) {  // one vector per step; vq == 0, compile-time offsets
      constexpr int v = rr / (P::CHV / P::NT);
      constexpr int toff = P::NT * (rr % (P::CHV / P::NT));
      f(v, r.tq + toff, r.hq + P::row(v) + (2 * toff / P::R) * P::WSTR);
    } else {  // NT / CHV vectors per step: the row skew difference is a runtime term
      constexpr int v = rr * (P::NT / P::CHV);
      const int vv = r.vq + v;
      f(vv, r.tq, r.hq + v * P::ROWA + P::skew(vv) - P::skew(r.vq));
    }
  });
}

// H (packed spectra, half pairs) -> global tile (natural order)
template <typename P>
__device__ __forceinline__ void p2_store(const P2Roles<P>& r, typename P::elem* dst, int nv) {
  using T = typename P::elem;
  p2_chunks<P>(r, [&](int vv, int t, const float2* h) {
    if (vv < nv) {
      const float4 f = *reinterpret_cast<const float4*>(h);
      T* d = dst + vv * P::N + 2 * t;
      gio<T>::st2(d, make_float2(f.x, f.z));
      gio<T>::st2(d + P::N / 2, make_float2(f.y, f.w));
    }
  });
}

// Spectral-resident weights: nvec packed fp32 spectra (rows of n, e.g. rdfft_fwd
// of w) copied into the half-pair layout the fused BCA kernels keep resident (dst rows row(v)).
template <typename P>
__device__ __forceinline__ void p2_load_spectra(float2* dst, const float* __restrict__ ws, int nvec, int lt,
                                                int nthr) {
  constexpr int N = P::N, HALF = N / 2;
  for (int e = lt; e < nvec * HALF; e += nthr) {
    const int v = e / HALF, hq = e % HALF;
    dst[P::hidx(v, hq)] = make_float2(__ldg(ws + (int64_t)v * N + hq), __ldg(ws + (int64_t)v * N + hq + HALF));
  }
}

// ---------------------------------------------------------------- inverse pieces
// staged tile (natural order) -> H half pairs
template <typename P>
__device__ __forceinline__ void p2_load(const P2Roles<P>& r, const typename P::elem* st, int nv, uint32_t k65536) {
  using T = typename P::elem;
  p2_chunks<P>(r, [&](int vv, int t, const float2* h) {
    if (vv < nv) {
      const T* src = st + vv * P::SROW + 2 * t;
      const float2 lo = sio<T>::ld2(src, k65536);
      const float2 hi = sio<T>::ld2(src + P::N / 2, k65536);
      *reinterpret_cast<float4*>(const_cast<float2*>(h)) = make_float4(lo.x, hi.x, lo.y, hi.y);
    }
  });
}

template <typename P>
__device__ __forceinline__ void p2_last_inv(const P2Roles<P>& r, int nv, int hoff = 0) {
  constexpr int M = P::M, WSTR = P::WSTR, LM = P::LM;
  if (r.v2 < nv) {
    // Y[q] is loaded into register rev(q); a DIT pass with conjugate twiddles then leaves
    // out[p] = M x IDFT(Y)[p] in register p, and Z'_j = IDFT(Y)[rev(j)] sits in register rev(j).
    float zr[M], zi[M];
    ct::static_for<0, M / 2>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      const float2 a = r.ha[hoff + q * WSTR];                    // (Re Y[q], -Im Y[q + M/2])
      const float2 bb = r.hm[hoff + (M / 2 - 1 - q) * WSTR];     // (Re Y[q + M/2], Im Y[q])
      zr[rev_bits<LM>(q)] = a.x;
      zi[rev_bits<LM>(q + M / 2)] = -a.y;
      zr[rev_bits<LM>(q + M / 2)] = bb.x;
      zi[rev_bits<LM>(q)] = bb.y;
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
      r.ha[hoff + jj * WSTR] = make_float2(zr[r1], zr[r2]);
      // k = R/2: the imaginary part (zero up to rounding) is dropped, so the pad keeps the exact
      // zero the next forward pass of the same buffer reads (fused BCA kernels reuse H per tile)
      if (!r.kz) r.hm[hoff + jj * WSTR] = make_float2(zi[r1], zi[r2]);
    });
  }
}

template <typename P>
__device__ __forceinline__ void p2_dc_inv(const P2Roles<P>& r, int nv, int hoff = 0) {
  constexpr int M = P::M, WSTR = P::WSTR;
  if (r.dv >= 0 && r.dv < nv) {
    float d[M];
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      const float2 a = r.hd[hoff + jj * WSTR];
      d[jj] = a.x;
      d[jj + M / 2] = a.y;
    });
    rfft_inv_reg<M>(d);
    ct::static_for<0, M / 2>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      r.hd[hoff + jj * WSTR] = make_float2(d[jj] * (1.0f / P::N), d[jj + M / 2] * (1.0f / P::N));
    });
  }
}

// inverse pass 1: H windows -> real signals in global memory
// acc: dst += result (the BCA forward's y += BCA(x) mode) instead of dst = result
template <typename P>
__device__ __forceinline__ void p2_pass1_inv(const P2Roles<P>& r, typename P::elem* dst_tile, int nv,
                                             bool acc = false, int hoff = 0) {
  using T = typename P::elem;
  constexpr int R = P::R, S = P::S;
  if (r.act1 && r.v1 < nv) {
    float2 b[R];
    ct::static_for<0, R / 2>([&](auto I) {
      constexpr int i = 2 * decltype(I)::value;
      const float4 f = *reinterpret_cast<const float4*>(r.h1 + hoff + i);
      b[i] = make_float2(f.x, f.y);
      b[i + 1] = make_float2(f.z, f.w);
    });
    rfft_inv_reg<R>(b);
    T* dst = dst_tile + r.s1;
    if (acc) {
      const uint32_t k65536 = kTwo16;
      ct::static_for<0, R>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const float2 o = gio<T>::ld2(dst + S * i, k65536);
        b[rev_bits<P::LR>(i)] = make_float2(b[rev_bits<P::LR>(i)].x + o.x, b[rev_bits<P::LR>(i)].y + o.y);
      });
    }
    ct::static_for<0, R>([&](auto I) {
      constexpr int i = decltype(I)::value;
      gio<T>::st2(dst + S * i, b[rev_bits<P::LR>(i)]);
    });
  }
}

// ---------------------------------------------------------------- TMA staging
template <typename T>
__device__ __forceinline__ void stage_issue(const T* src, uint32_t bytes, void* dst, uint64_t* bar) {
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(bar, bytes);
  bulk_g2s(dst, src, bytes, bar);
}
// nrows rows of n elements -> staged rows of SROW elements (one bulk copy per row)
template <typename P>
__device__ __forceinline__ void stage_issue_rows(const typename P::elem* src, int nrows, void* dst, uint64_t* bar) {
  using T = typename P::elem;
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(bar, (uint32_t)(nrows * P::N * (int)sizeof(T)));
  for (int v = 0; v < nrows; ++v)
    bulk_g2s(reinterpret_cast<T*>(dst) + v * P::SROW, src + (int64_t)v * P::N, (uint32_t)(P::N * sizeof(T)), bar);
}

// ---------------------------------------------------------------- rdfft kernels
template <typename P>
struct P2Smem {  // [stage 0 .. NSTG-1][H][TW][bars]
  static constexpr size_t H_OFF = (size_t)P::NSTG * P::STAGE;
  static constexpr size_t TW_OFF = H_OFF + (size_t)P::HF * 8;
  static constexpr size_t BAR_OFF = TW_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BYTES = BAR_OFF + 8 * (P::NSTG > 0 ? P::NSTG : 1);
};

template <typename P, bool kInv>
__global__ void __launch_bounds__(P::NTT) rdfft2_kernel(typename P::elem* __restrict__ x, int64_t batch) {
  using T = typename P::elem;
  using L = P2Smem<P>;
  constexpr int VT = P::VT, N = P::N;
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float2* H = reinterpret_cast<float2*>(base + L::H_OFF);
  float2* TW = reinterpret_cast<float2*>(base + L::TW_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  const int tid = threadIdx.x;
  p2_tables<P>(kInv ? nullptr : TW, kInv ? TW : nullptr, tid, P::NTT);
  if (!kInv) p2_zero_pads<P>(H, VT, tid, P::NTT);
  if (tid == 0) {
    for (int q = 0; q < (P::NSTG > 0 ? P::NSTG : 1); ++q) mbar_init(bar + q, 1);
    fence_mbar_init();
  }
  const P2Roles<P> r(H, TW, TW, tid);
  const uint32_t k65536 = kTwo16;
  const int64_t ntiles = (batch + VT - 1) / VT;
  auto tile_rows = [&](int64_t t) { return (int)(batch - t * VT < VT ? batch - t * VT : VT); };
  __syncthreads();
  constexpr int NS = P::NSTG;
  static_assert(!(kInv && NS == 0), "the inverse transform stages its input");
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) {
      const int64_t t = blockIdx.x + (int64_t)q * gridDim.x;
      if (t < ntiles) stage_issue_rows<P>(x + t * VT * (int64_t)N, tile_rows(t), base + q * P::STAGE, bar + q);
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int nv = (int)(batch - tile * VT < VT ? batch - tile * VT : VT);
    T* xt = x + tile * VT * (int64_t)N;
    if constexpr (NS == 0) {  // forward without staging: pass 1 loads straight from HBM
      p2_pass1_fwd<P, true>(r, xt, nv, k65536);
      __syncthreads();
      if constexpr (P::FD) {
        p2_last_fwd_direct<P>(r, xt, nv);
        p2_dc_fwd_direct<P>(r, xt, nv);
      } else {
        p2_last_fwd<P>(r, nv);
        p2_dc_fwd<P>(r, nv);
        __syncthreads();
        p2_store<P>(r, xt, nv);
      }
    } else {
      const int sb = it % NS;
      const T* st = reinterpret_cast<const T*>(base + sb * P::STAGE);
      const int64_t nxt = tile + NS * (int64_t)gridDim.x;
      mbar_wait(bar + sb, (it / NS) & 1);
      if (!kInv) {
        p2_pass1_fwd<P>(r, st, nv, k65536);
        __syncthreads();  // H complete; staging buffer sb consumed
        if (tid == 0 && nxt < ntiles) stage_issue_rows<P>(x + nxt * VT * (int64_t)N, tile_rows(nxt), base + sb * P::STAGE, bar + sb);
        if constexpr (P::FD) {
          p2_last_fwd_direct<P>(r, xt, nv);
          p2_dc_fwd_direct<P>(r, xt, nv);
        } else {
          p2_last_fwd<P>(r, nv);
          p2_dc_fwd<P>(r, nv);
          __syncthreads();
          if (P::NTT == P::NT || tid < P::NT) p2_store<P>(r, xt, nv);
        }
      } else {
        p2_load<P>(r, st, nv, k65536);
        __syncthreads();
        if (tid == 0 && nxt < ntiles) stage_issue_rows<P>(x + nxt * VT * (int64_t)N, tile_rows(nxt), base + sb * P::STAGE, bar + sb);
        p2_last_inv<P>(r, nv);
        p2_dc_inv<P>(r, nv);
        __syncthreads();
        p2_pass1_inv<P>(r, xt, nv);
      }
    }
    __syncthreads();  // H free for the next tile
  }
}

template <typename P, bool kInv>
bool launch_plan2_dir(typename P::elem* x, int64_t batch, int sms, cudaStream_t st) {
  using L = P2Smem<P>;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  auto k = rdfft2_kernel<P, kInv>;
  static int per_sm_dev[kMaxDevices] = {};
  int& per_sm = per_sm_dev[device_index()];
  if (!per_sm) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, P::NTT, L::BYTES);
    if (per_sm < 1) per_sm = 1;
    if (verbose())
      std::fprintf(stderr, "[rdfft] plan2 n=%d R=%d VT=%d NSTG=%d inv=%d: %zu B smem, %d threads, %d CTAs/SM\n", P::N,
                   P::R, P::VT, P::NSTG, (int)kInv, (size_t)L::BYTES, P::NTT, per_sm);
  }
  const int64_t tiles = (batch + P::VT - 1) / P::VT;
  const int grid = (int)(tiles < (int64_t)per_sm * sms ? tiles : (int64_t)per_sm * sms);
  k<<<grid, P::NTT, L::BYTES, st>>>(x, batch);
  return true;
}

// ---------------------------------------------------------------- forward with an output tile
// The last pass and the DC lanes write the packed outputs (element type T, RNE for bf16) into an
// output staging tile O in natural order; one thread then stores O's rows with TMA bulk copies
// (cp.async.bulk shared -> global).  Against rdfft2_kernel this drops the H -> HBM store phase
// (a fp32 read of H per element plus the STG instructions) for one narrow shared store per element,
// and the outputs reach HBM as whole contiguous rows.  O is reused per tile once the previous
// tile's bulk store has read it (cp.async.bulk.wait_group.read before the barrier that precedes
// the last pass).  NSTG = 0: pass 1 reads HBM directly (no input staging buffer).
// O row skew (bytes, 16-byte multiples for the bulk copies): the two interleaved vectors of an
// R = 32 warp (16 lanes x 2 B each) fall on disjoint banks and the 8 DC lanes (one per vector) on 8
// distinct banks at a stride of 20 words (bf16); R = 16 (4 vectors of 8 lanes per warp) uses 12
// words; fp32 rows are 16 lanes x 4 B, so 16 words.
template <typename P>
struct P2fSmem {
  using T = typename P::elem;
  static constexpr int OSKEWB = sizeof(T) == 2 ? (P::R == 32 ? 80 : 48) : (P::R == 32 ? 64 : 32);
  static constexpr int OROW = P::N + OSKEWB / (int)sizeof(T);
  static constexpr size_t O_OFF = (size_t)P::NSTG * P::STAGE;
  static constexpr size_t H_OFF = O_OFF + (size_t)P::VT * OROW * sizeof(T);
  static constexpr size_t TW_OFF = H_OFF + (size_t)P::HF * 8;
  static constexpr size_t BAR_OFF = TW_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BYTES = BAR_OFF + 8 * (P::NSTG > 0 ? P::NSTG : 1);
  static_assert((OROW * sizeof(T)) % 16 == 0 && O_OFF % 16 == 0, "O rows must be 16-byte aligned (bulk copies)");
};

template <typename P>
__global__ void __launch_bounds__(P::NT) rdfft2fo_kernel(typename P::elem* __restrict__ x, int64_t batch) {
  using T = typename P::elem;
  using L = P2fSmem<P>;
  constexpr int VT = P::VT, N = P::N, NS = P::NSTG;
  static_assert(NS <= 1, "one input staging buffer (or none)");
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  T* O = reinterpret_cast<T*>(base + L::O_OFF);
  float2* H = reinterpret_cast<float2*>(base + L::H_OFF);
  float2* TW = reinterpret_cast<float2*>(base + L::TW_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  const int tid = threadIdx.x;
  p2_tables<P>(TW, nullptr, tid, P::NT);
  p2_zero_pads<P>(H, VT, tid, P::NT);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  const P2Roles<P> r(H, TW, TW, tid);
  const uint32_t k65536 = kTwo16;
  const int64_t ntiles = (batch + VT - 1) / VT;
  auto tile_rows = [&](int64_t t) { return (int)(batch - t * VT < VT ? batch - t * VT : VT); };
  __syncthreads();
  if (NS > 0 && tid == 0 && (int64_t)blockIdx.x < ntiles)
    stage_issue_rows<P>(x + (int64_t)blockIdx.x * VT * N, tile_rows(blockIdx.x), base, bar);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int nv = tile_rows(tile);
    T* xt = x + tile * VT * (int64_t)N;
    if constexpr (NS > 0) {
      mbar_wait(bar, it & 1);
      p2_pass1_fwd<P>(r, reinterpret_cast<const T*>(base), nv, k65536);
    } else {
      p2_pass1_fwd<P, true>(r, xt, nv, k65536);
    }
    if (tid == 0) bulk_wait_read<0>();  // the previous tile's bulk store has read O
    __syncthreads();                    // H complete; staging buffer consumed; O free
    const int64_t nxt = tile + gridDim.x;
    if (NS > 0 && tid == 0 && nxt < ntiles) stage_issue_rows<P>(x + nxt * VT * (int64_t)N, tile_rows(nxt), base, bar);
    p2_last_fwd_direct<P, sst1<T>, L::OROW>(r, O, nv);
    p2_dc_fwd_direct<P, sst1<T>, L::OROW>(r, O, nv);
    fence_proxy_async_smem();  // O's generic-proxy writes before the bulk store reads them
    __syncthreads();           // O complete; H free for the next tile
    if (tid == 0) {
      for (int v = 0; v < nv; ++v) bulk_s2g(xt + (int64_t)v * N, O + v * L::OROW, (uint32_t)(N * sizeof(T)));
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait<0>();
}

template <typename P>
bool launch_plan2fo(typename P::elem* x, int64_t batch, int sms, cudaStream_t st) {
  using L = P2fSmem<P>;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  auto k = rdfft2fo_kernel<P>;
  static int per_sm_dev[kMaxDevices] = {};
  int& per_sm = per_sm_dev[device_index()];
  if (!per_sm) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, P::NT, L::BYTES);
    if (per_sm < 1) per_sm = 1;
    if (verbose())
      std::fprintf(stderr, "[rdfft] plan2fo n=%d R=%d VT=%d NSTG=%d: %zu B smem, %d threads, %d CTAs/SM\n", P::N, P::R,
                   P::VT, P::NSTG, (size_t)L::BYTES, P::NT, per_sm);
  }
  const int64_t tiles = (batch + P::VT - 1) / P::VT;
  const int grid = (int)(tiles < (int64_t)per_sm * sms ? tiles : (int64_t)per_sm * sms);
  k<<<grid, P::NT, L::BYTES, st>>>(x, batch);
  return true;
}

// forward plan PF, inverse plan PI (may differ in staging depth)
template <typename PF, typename PI>
bool launch_plan2(typename PF::elem* x, int64_t batch, bool inverse, int sms, cudaStream_t st) {
  return inverse ? launch_plan2_dir<PI, true>(x, batch, sms, st) : launch_plan2_dir<PF, false>(x, batch, sms, st);
}

}  // namespace rdfft
