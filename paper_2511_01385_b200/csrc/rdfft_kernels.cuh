// rdfft_kernels.cuh — register-blocked in-place rdFFT kernels for sm_100a.
//
// Plan "2-pass" for n = R * M (R, M powers of two, M <= R):
//
//  pass 1 (stages m = 1 .. R/2 of the paper's schedule):
//    After bit reversal, the first log2 R stages act independently on windows
//    of R consecutive slots; window w holds the packed R-point spectrum of the
//    decimated subsequence x[rev(w) :: n/R] (per-stage invariant, Eq. 6).  So
//    thread c loads two decimated subsequences x[2c + S i], x[2c+1 + S i]
//    (S = n/R; one 4-byte bf16x2 / 8-byte float2 global load per i, coalesced
//    across c), runs the paper's stages in registers with compile-time
//    twiddles, and writes windows rev(2c) and rev(2c) + S/2.
//
//  last pass (stages m = R .. n/2): by Prop. 1 the four-slot groups of these
//    log2 M stages close over S_k = {j R +- k} (the "register-blocking closure"
//    of SURVEY §0 fact 4), so one thread owns S_k and finishes all remaining
//    stages without exchange.  For 1 <= k < R/2 the t = log2 M stages are
//    regrouped as a twiddle W_n^{k rev(j)} on the M block spectra Z_j(k)
//    followed by an M-point complex DIT FFT (the same radix-2 butterflies,
//    reordered); S_0 (the DC / Nyquist slots of every block) runs a real
//    M-point FFT plus an odd-frequency M-point FFT in a dedicated warp.
//
//  The intermediate lives in shared memory as fp32 "half pairs"
//  H[q] = (slot q, slot q + n/2): every shared access is 8 or 16 bytes, and
//  both halves share twiddles in pass 1.  Output (forward) / input (inverse)
//  goes through H with fully coalesced 128-byte-per-warp global accesses.
//  Global memory is touched exactly once per element in each direction and
//  nothing outside the vector is read or written (in place, zero scratch).
//
// The inverse kernel runs the reversed graph (Eq. 7): last pass
// first (conjugate twiddles, DIF), then pass 1 with the paper's inverse stages;
// 1/n is folded into the last pass's twiddle table (reading C4).
#pragma once

#include "common.cuh"
#include "regfft.cuh"

namespace rdfft {

template <typename T>
struct sio;  // shared-memory pair loads of T
template <>
struct sio<float> {
  __device__ __forceinline__ static float2 ld2(const float* p, uint32_t) {
    return *reinterpret_cast<const float2*>(p);
  }
};

// 2^16 as a constant-bank operand ptxas cannot fold (see sio<__nv_bfloat16>::ld2).
__constant__ uint32_t kTwo16 = 65536u;
template <>
struct sio<__nv_bfloat16> {
  // k65536 must be an opaque register: u * k65536 (= u << 16) then issues as IMAD on the
  // full-rate FMA pipe instead of SHF on the half-rate ALU pipe.
  __device__ __forceinline__ static float2 ld2(const __nv_bfloat16* p, uint32_t k65536) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    return make_float2(__uint_as_float(u * k65536), __uint_as_float(u & 0xffff0000u));
  }
};

template <typename T>
struct gio;
template <>
struct gio<float> {
  using pair_t = float2;
  __device__ __forceinline__ static float2 ld2(const float* p) { return __ldcs(reinterpret_cast<const float2*>(p)); }
  __device__ __forceinline__ static void st2(float* p, float2 v) { __stcs(reinterpret_cast<float2*>(p), v); }
};
template <>
struct gio<__nv_bfloat16> {
  __device__ __forceinline__ static float2 ld2(const __nv_bfloat16* p) {
    const uint32_t u = __ldcs(reinterpret_cast<const unsigned int*>(p));
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
  }
  __device__ __forceinline__ static void st2(__nv_bfloat16* p, float2 v) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
    __stcs(reinterpret_cast<unsigned int*>(p), *reinterpret_cast<unsigned int*>(&h));
  }
};

template <typename T, int N, int R, int VT>
struct Plan2 {
  static constexpr int LN = ilog2c<N>();
  static constexpr int LR = ilog2c<R>();
  static constexpr int M = N / R;           // last-pass FFT size (blocks per vector)
  static constexpr int LM = ilog2c<M>();
  static constexpr int S = N / R;           // decimated subsequences per vector
  static constexpr int LS = ilog2c<S>();
  static constexpr int P1 = S / 2;          // pass-1 threads per vector
  static constexpr int LPV = R / 2;         // last-pass lanes per vector: k = 1 .. R/2
  static constexpr int NT = VT * LPV;
  static constexpr int WSTR = R + 2;        // float2 per window + 16 B pad (conflict-free window writes)
  static constexpr int ROWF = (N / (2 * R)) * WSTR + 2;  // float2 per vector row of H (+16 B skew)
  static constexpr int TWF = M * LPV;
  static constexpr int CHV = N / 4;         // 16-byte H chunks per vector (store / load phase)
  static constexpr int CPT = VT * CHV / NT; // chunks per thread per tile
  static constexpr int STAGE = VT * N * (int)sizeof(T);  // bytes per staging buffer
  static constexpr size_t SMEM = 2 * (size_t)STAGE + (size_t)(VT * ROWF + TWF) * 8 + 16;
  static_assert(M <= R && M >= 4 && R == 32 && S >= 16, "2-pass plan shape");
  static_assert(NT % 32 == 0 && VT * P1 <= NT, "thread mapping");
  static_assert(ROWF % 16 == 2, "rows skewed by 16 B: the DC-set warp (lanes = vectors) is conflict-free");
  static_assert(VT <= 32, "one DC-set lane per vector in the last warp");
  static_assert(CHV % NT == 0 || NT % CHV == 0, "store-phase mapping");
};

// Shared memory (bytes): [stage 0][stage 1] (T, natural order, filled by cp.async.bulk)
//   H[v * ROWF + w * WSTR + i] (float2) = (slot w R + i, slot w R + i + N/2), w < S/2, i < R;
//     H[v * ROWF + w * WSTR + R] = 0: the zero imaginary input of the k = R/2 lane (forward)
//     or the sink of its discarded imaginary output (inverse).
//   TW[j * LPV + k - 1] = W_N^{k rev(j)} (forward) | conj(W_N^{k rev(j)}) / N (inverse)
//   two mbarriers (one per staging buffer).
template <typename P, bool kInv>
__device__ __forceinline__ void plan2_init(float2* H, float2* TW, uint64_t* bar) {
  constexpr int N = P::M * 32;
  for (int e = threadIdx.x; e < P::TWF; e += P::NT) {
    const int j = e / P::LPV, k = 1 + e % P::LPV;
    float s, c;
    sincospif(2.0f * (float)(k * rev_bits<P::LM>(j)) / (float)N, &s, &c);
    TW[e] = kInv ? make_float2(c * (1.0f / N), s * (1.0f / N)) : make_float2(c, -s);
  }
  for (int e = threadIdx.x; e < (P::ROWF / P::WSTR) * (P::NT / P::LPV); e += P::NT) {
    float2* pad = H + (e / (P::ROWF / P::WSTR)) * P::ROWF + (e % (P::ROWF / P::WSTR)) * P::WSTR + 32;
    pad[0] = make_float2(0.f, 0.f);
    pad[1] = make_float2(0.f, 0.f);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
}

template <typename P, typename T>
__device__ __forceinline__ void plan2_issue(T* x, int64_t batch, int64_t tile, unsigned char* stage, uint64_t* bar) {
  constexpr int VT = P::NT / P::LPV, N = P::M * 32;
  const int64_t nv = batch - tile * VT < VT ? batch - tile * VT : VT;
  const uint32_t bytes = (uint32_t)(nv * N * (int)sizeof(T));
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(bar, bytes);
  bulk_g2s(stage, x + tile * VT * (int64_t)N, bytes, bar);
}

// Visit this thread's store/load-phase chunks: f(v, t_off, h_off) with chunk t = tid-part + t_off of
// vector v (compile-time parts) and h_off its H float2 offset relative to the per-thread base.
template <typename P, typename F>
__device__ __forceinline__ void plan2_chunks(F&& f) {
  ct::static_for<0, P::CPT>([&](auto RR) {
    constexpr int r = decltype(RR)::value;
    if constexpr (P::CHV % P::NT == 0) {
      constexpr int v = r / (P::CHV / P::NT);
      constexpr int toff = P::NT * (r % (P::CHV / P::NT));
      f(v, toff, v * P::ROWF + (2 * toff / 32) * P::WSTR);
    } else {
      constexpr int v = r * (P::NT / P::CHV);
      f(v, 0, v * P::ROWF);
    }
  });
}

// ------------------------------------------------------------------ forward
template <typename T, int N, int R, int VT>
__global__ void __launch_bounds__(Plan2<T, N, R, VT>::NT) rdfft_fwd2_kernel(T* __restrict__ x, int64_t batch) {
  using P = Plan2<T, N, R, VT>;
  constexpr int M = P::M, S = P::S, WSTR = P::WSTR;
  extern __shared__ float4 smem4[];
  unsigned char* stage = reinterpret_cast<unsigned char*>(smem4);
  float2* H = reinterpret_cast<float2*>(stage + 2 * P::STAGE);
  float2* TW = H + VT * P::ROWF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(TW + P::TWF);
  plan2_init<P, false>(H, TW, bar);
  const int tid = threadIdx.x;
  // pass-1 role: vector v1, window w1 (lane order = window order), subsequences 2c1, 2c1+1
  const int v1 = tid / P::P1, w1 = tid % P::P1;
  const int c1 = rev_bits<P::LS - 1>(w1);  // rev_LS(2 c1) == w1
  const bool act1 = tid < VT * P::P1;
  float2* h1 = H + v1 * P::ROWF + w1 * WSTR;
  const int s1 = v1 * N + 2 * c1;  // element offset in the staging tile
  // last-pass role: vector v2, set k
  const int v2 = tid / P::LPV, k = 1 + tid % P::LPV;
  float2* ha = H + v2 * P::ROWF + k;                                   // slots j R + k
  float2* hm = H + v2 * P::ROWF + (R - k);                             // slots (j+1) R - k
  const float2* hmi = (k == R / 2) ? (H + v2 * P::ROWF + R) : hm;      // k = R/2: zero imaginary input
  const float2* tw = TW + (k - 1);
  const int dv = tid - (P::NT - 32);  // DC-set role: lane dv of the last warp owns vector dv
  float2* hd = H + dv * P::ROWF;                                       // slots j R (block DCs)
  // store role: chunk (slots 2t, 2t+1 | +N/2), t = tid-part + compile-time offsets
  const int tq = (P::CHV % P::NT == 0) ? tid : tid % P::CHV;
  const int vq = (P::CHV % P::NT == 0) ? 0 : tid / P::CHV;
  const float2* hq = H + vq * P::ROWF + (2 * tq / R) * WSTR + (2 * tq) % R;
  const int64_t ntiles = (batch + VT - 1) / VT;
  const uint32_t k65536 = kTwo16;
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < 2; ++q) {
      const int64_t t = blockIdx.x + (int64_t)q * gridDim.x;
      if (t < ntiles) plan2_issue<P>(x, batch, t, stage + q * P::STAGE, bar + q);
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int nv = (int)(batch - tile * VT < VT ? batch - tile * VT : VT);
    T* xt = x + tile * VT * (int64_t)N;
    const int sb = it & 1;
    const T* st = reinterpret_cast<const T*>(stage + sb * P::STAGE);
    mbar_wait(bar + sb, (it >> 1) & 1);
    // ---------------- pass 1: two decimated subsequences -> two packed R-point spectra
    if (act1 && v1 < nv) {
      float2 b[R];
      ct::static_for<0, R>([&](auto I) {
        constexpr int i = decltype(I)::value;
        b[rev_bits<P::LR>(i)] = sio<T>::ld2(st + s1 + S * i, k65536);
      });
      rfft_fwd_reg<R>(b);
      ct::static_for<0, R / 2>([&](auto I) {
        constexpr int i = 2 * decltype(I)::value;
        *reinterpret_cast<float4*>(h1 + i) = make_float4(b[i].x, b[i].y, b[i + 1].x, b[i + 1].y);
      });
    }
    __syncthreads();  // H complete; staging buffer sb consumed
    if (tid == 0 && tile + 2 * (int64_t)gridDim.x < ntiles)
      plan2_issue<P>(x, batch, tile + 2 * (int64_t)gridDim.x, stage + sb * P::STAGE, bar + sb);
    // ---------------- last pass: set S_k, k = 1 .. R/2
    if (v2 < nv) {
      float zr[M], zi[M];
      ct::static_for<0, M / 2>([&](auto J) {
        constexpr int jj = decltype(J)::value;
        const float2 a = ha[jj * WSTR];
        const float2 bb = hmi[jj * WSTR];
        zr[jj] = a.x;
        zr[jj + M / 2] = a.y;
        zi[jj] = bb.x;
        zi[jj + M / 2] = bb.y;
      });
      ct::static_for<1, M>([&](auto J) {
        constexpr int j = decltype(J)::value;
        const float2 t = tw[j * P::LPV];
        const float r = zr[j];
        zr[j] = fmaf(r, t.x, -zi[j] * t.y);
        zi[j] = fmaf(r, t.y, zi[j] * t.x);
      });
      cfft_dit<M>(zr, zi);
      ct::static_for<0, M / 2>([&](auto Q) {
        constexpr int q = decltype(Q)::value;
        ha[q * WSTR] = make_float2(zr[q], -zi[q + M / 2]);
        hm[(M / 2 - 1 - q) * WSTR] = make_float2(zr[q + M / 2], zi[q]);
      });
    }
    if (dv >= 0 && dv < nv) {  // block DCs j R: packed real M-point DFT (input already bit-reversed)
      float d[M];
      ct::static_for<0, M / 2>([&](auto J) {
        constexpr int jj = decltype(J)::value;
        const float2 a = hd[jj * WSTR];
        d[jj] = a.x;
        d[jj + M / 2] = a.y;
      });
      rfft_fwd_reg<M>(d);
      ct::static_for<0, M / 2>([&](auto J) {
        constexpr int jj = decltype(J)::value;
        hd[jj * WSTR] = make_float2(d[jj], d[jj + M / 2]);
      });
    }
    __syncthreads();
    // ---------------- store: chunk = slots (2t, 2t+1) and (2t + N/2, 2t+1 + N/2)
    plan2_chunks<P>([&](int v, int toff, int hoff) {
      if (vq + v < nv) {
        const float4 f = *reinterpret_cast<const float4*>(hq + hoff);
        T* dst = xt + (vq + v) * N + 2 * (tq + toff);
        gio<T>::st2(dst, make_float2(f.x, f.z));
        gio<T>::st2(dst + N / 2, make_float2(f.y, f.w));
      }
    });
    __syncthreads();  // H free for the next tile
  }
}

// ------------------------------------------------------------------ inverse
template <typename T, int N, int R, int VT>
__global__ void __launch_bounds__(Plan2<T, N, R, VT>::NT) rdfft_inv2_kernel(T* __restrict__ x, int64_t batch) {
  using P = Plan2<T, N, R, VT>;
  constexpr int M = P::M, S = P::S, WSTR = P::WSTR;
  extern __shared__ float4 smem4[];
  unsigned char* stage = reinterpret_cast<unsigned char*>(smem4);
  float2* H = reinterpret_cast<float2*>(stage + 2 * P::STAGE);
  float2* TW = H + VT * P::ROWF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(TW + P::TWF);
  plan2_init<P, true>(H, TW, bar);
  const int tid = threadIdx.x;
  const int v1 = tid / P::P1, w1 = tid % P::P1;
  const int c1 = rev_bits<P::LS - 1>(w1);
  const bool act1 = tid < VT * P::P1;
  const float2* h1 = H + v1 * P::ROWF + w1 * WSTR;
  const int v2 = tid / P::LPV, k = 1 + tid % P::LPV;
  float2* ha = H + v2 * P::ROWF + k;
  float2* hm = H + v2 * P::ROWF + (R - k);
  float2* hmo = (k == R / 2) ? (H + v2 * P::ROWF + R) : hm;  // k = R/2: discard imaginary output
  const float2* tw = TW + (k - 1);
  const int dv = tid - (P::NT - 32);
  float2* hd = H + dv * P::ROWF;
  const int tq = (P::CHV % P::NT == 0) ? tid : tid % P::CHV;
  const int vq = (P::CHV % P::NT == 0) ? 0 : tid / P::CHV;
  float2* hq = H + vq * P::ROWF + (2 * tq / R) * WSTR + (2 * tq) % R;
  const int64_t ntiles = (batch + VT - 1) / VT;
  const uint32_t k65536 = kTwo16;
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < 2; ++q) {
      const int64_t t = blockIdx.x + (int64_t)q * gridDim.x;
      if (t < ntiles) plan2_issue<P>(x, batch, t, stage + q * P::STAGE, bar + q);
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int nv = (int)(batch - tile * VT < VT ? batch - tile * VT : VT);
    T* xt = x + tile * VT * (int64_t)N;
    const int sb = it & 1;
    const T* st = reinterpret_cast<const T*>(stage + sb * P::STAGE);
    mbar_wait(bar + sb, (it >> 1) & 1);
    // ---------------- packed spectra (staging, natural order) -> H half pairs
    plan2_chunks<P>([&](int v, int toff, int hoff) {
      if (vq + v < nv) {
        const T* src = st + (vq + v) * N + 2 * (tq + toff);
        const float2 lo = sio<T>::ld2(src, k65536);
        const float2 hi = sio<T>::ld2(src + N / 2, k65536);
        *reinterpret_cast<float4*>(hq + hoff) = make_float4(lo.x, hi.x, lo.y, hi.y);
      }
    });
    __syncthreads();
    if (tid == 0 && tile + 2 * (int64_t)gridDim.x < ntiles)
      plan2_issue<P>(x, batch, tile + 2 * (int64_t)gridDim.x, stage + sb * P::STAGE, bar + sb);
    // ---------------- inverse last pass
    if (v2 < nv) {
      float zr[M], zi[M];
      // Y[q] is loaded into register rev(q); a DIT pass with conjugate twiddles then leaves
      // out[p] = M x IDFT(Y)[p] in register p, and Z'_j = IDFT(Y)[rev(j)] sits in register rev(j).
      constexpr int LM = P::LM;
      ct::static_for<0, M / 2>([&](auto Q) {
        constexpr int q = decltype(Q)::value;
        const float2 a = ha[q * WSTR];                    // (Re Y[q], -Im Y[q + M/2])
        const float2 bb = hm[(M / 2 - 1 - q) * WSTR];     // (Re Y[q + M/2], Im Y[q])
        zr[rev_bits<LM>(q)] = a.x;
        zi[rev_bits<LM>(q + M / 2)] = -a.y;
        zr[rev_bits<LM>(q + M / 2)] = bb.x;
        zi[rev_bits<LM>(q)] = bb.y;
      });
      cfft_dit<M, true>(zr, zi);
      ct::static_for<0, M>([&](auto J) {
        constexpr int j = decltype(J)::value;
        constexpr int rj = rev_bits<LM>(j);
        const float2 t = tw[j * P::LPV];
        const float r = zr[rj];
        zr[rj] = fmaf(r, t.x, -zi[rj] * t.y);
        zi[rj] = fmaf(r, t.y, zi[rj] * t.x);
      });
      ct::static_for<0, M / 2>([&](auto J) {
        constexpr int jj = decltype(J)::value;
        constexpr int r1 = rev_bits<P::LM>(jj), r2 = rev_bits<P::LM>(jj + M / 2);
        ha[jj * WSTR] = make_float2(zr[r1], zr[r2]);
        hmo[jj * WSTR] = make_float2(zi[r1], zi[r2]);
      });
    }
    if (dv >= 0 && dv < nv) {  // block DCs: inverse packed real M-point DFT
      float d[M];
      ct::static_for<0, M / 2>([&](auto J) {
        constexpr int jj = decltype(J)::value;
        const float2 a = hd[jj * WSTR];
        d[jj] = a.x;
        d[jj + M / 2] = a.y;
      });
      rfft_inv_reg<M>(d);
      ct::static_for<0, M / 2>([&](auto J) {
        constexpr int jj = decltype(J)::value;
        hd[jj * WSTR] = make_float2(d[jj] * (1.0f / N), d[jj + M / 2] * (1.0f / N));
      });
    }
    __syncthreads();
    // ---------------- inverse pass 1 -> global
    if (act1 && v1 < nv) {
      float2 b[R];
      ct::static_for<0, R / 2>([&](auto I) {
        constexpr int i = 2 * decltype(I)::value;
        const float4 f = *reinterpret_cast<const float4*>(h1 + i);
        b[i] = make_float2(f.x, f.y);
        b[i + 1] = make_float2(f.z, f.w);
      });
      rfft_inv_reg<R>(b);
      T* dst = xt + v1 * N + 2 * c1;
      ct::static_for<0, R>([&](auto I) {
        constexpr int i = decltype(I)::value;
        gio<T>::st2(dst + S * i, b[rev_bits<P::LR>(i)]);
      });
    }
    __syncthreads();  // H free for the next tile
  }
}

// ------------------------------------------------------------------ dispatch
template <typename T, int N, int R, int VT>
bool launch_plan2(T* x, int64_t batch, bool inverse, int sms, cudaStream_t st) {
  using P = Plan2<T, N, R, VT>;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  auto kf = rdfft_fwd2_kernel<T, N, R, VT>;
  auto ki = rdfft_inv2_kernel<T, N, R, VT>;
  static bool configured = false;
  static int per_sm = 1;
  if (!configured) {
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    cudaFuncSetAttribute(ki, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(ki, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, kf, P::NT, P::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ki, P::NT, P::SMEM);
    per_sm = a < b ? a : b;
    if (per_sm < 1) per_sm = 1;
    configured = true;
  }
  const int64_t tiles = (batch + VT - 1) / VT;
  const int grid = (int)(tiles < (int64_t)per_sm * sms ? tiles : (int64_t)per_sm * sms);
  if (inverse)
    ki<<<grid, P::NT, P::SMEM, st>>>(x, batch);
  else
    kf<<<grid, P::NT, P::SMEM, st>>>(x, batch);
  return true;
}

// Returns true when a specialised kernel was launched for (n, T).
template <typename T>
bool launch_rdfft_fast(T* x, int64_t batch, int n, int logn, bool inverse, int sms, cudaStream_t st) {
  (void)logn;
  switch (n) {
    case 512: return launch_plan2<T, 512, 32, 8>(x, batch, inverse, sms, st);
    case 1024: return launch_plan2<T, 1024, 32, 8>(x, batch, inverse, sms, st);
    default: return false;
  }
}

}  // namespace rdfft
