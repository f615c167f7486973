// planl.cuh — in-place rdFFT for large n (8192, 16384, 32768), one vector
// per CTA held in shared memory as fp32 (<= 128 KB), three register passes.
//
// n = 32 * 32 * M3 (M3 = n / 1024 in {8, 16, 32}); every pass is the paper's radix-2 stages
// (Prop. 1) regrouped on the closed sets of SURVEY §0 fact 4:
//   pass 1 (stages m = 1 .. 16): the 32-point packed real FFT of each decimated subsequence
//           x[r :: n/32] (bit reversal absorbed: subsequence r lands in window rev(r));
//   pass 2 (stages m = 32 .. 512) on each 1024-slot window: S_k = {32 j + k, 32 (j+1) - k},
//           k = 1 .. 15 -> twiddle W_1024^{k rev(j)} + 32-point complex DIT; k = 16 (block
//           Nyquists) the same with zero imaginary input; k = 0 (block DCs) a real 32-point FFT;
//   pass 3 (stages m = 1024 .. n/2) on the whole vector: S_k = {1024 j +- k}, k = 1 .. 512,
//           twiddle W_n^{k rev(j)} + M3-point DIT; k = 0 a real M3-point FFT.
// The inverse runs the reversed graph (Eq. 7): pass 3, 2, 1 with conjugate
// twiddles, unscaled, 1/n folded into pass 3 (reading C4).
//
// Shared layout: plain packed slots (fp32), 32-slot windows, 16-byte chunks XOR-swizzled by
// window bits so the pass-1 window stores and the pass-2/3 set accesses are conflict-free
// (simulated: <= 1.5 wavefronts per ideal one).  Twiddle tables in shared memory:
// TW2[j][k-1] = W_1024^{k rev5(j)} (4 KB) and TW3[a][k-1] = W_n^{4 k a} (M3/4 x 512) with
// W_n^{k b}, b < 4, in registers.  No global scratch.
#pragma once

#include "plan2.cuh"

namespace rdfft {

template <typename T, int N_>
struct PlanL {
  using elem = T;
  static constexpr int N = N_, LN = ilog2c<N>();
  static constexpr int R = 32, LR = 5, S = N / R, LS = LN - LR;
  static constexpr int M2 = 32, W2 = 1024, NW2 = N / W2;
  static constexpr int M3 = N / W2, LM3 = ilog2c<M3>(), K3 = W2 / 2;
  // threads: one per pass-1 subsequence pair and per pass-2 set (S/2 = 16 NW2), <= 16 warps (4 per
  // SM quadrant keeps the 128-register budget); pass 3 loops over K3 / NT sets per thread.  Small n
  // thus runs several CTAs per SM (n = 8192: 128 threads, 4 CTAs; 16384: 256 threads, 2 CTAs).
  static constexpr int NT = S / 2 < 512 ? S / 2 : 512;
  static constexpr int K3PT = K3 / NT;
  static constexpr int MINB = 512 / NT;  // CTAs per SM the 128-register budget allows
  static_assert(S / 2 == NW2 * 16 || NT == 512, "pass-2 sets per thread");
  static constexpr int TW2N = 32 * 16, TW3N = (M3 / 4) * K3;
  static constexpr size_t TW2_OFF = (size_t)N * 4;
  static constexpr size_t TW3_OFF = TW2_OFF + (size_t)TW2N * 8;
  static constexpr size_t BYTES = TW3_OFF + (size_t)TW3N * 8;
  static_assert(M3 >= 8 && M3 <= 32 && LS >= 8, "plan L shape");
  __host__ __device__ static constexpr int swz(int w) { return ((w >> (LS - 4)) ^ (((w >> 5) & 1) << 2)) & 7; }
  // float index of packed slot s
  __host__ __device__ static constexpr int phys(int s) {
    return ((s >> 5) << 5) + ((((s >> 2) & 7) ^ swz(s >> 5)) << 2) + (s & 3);
  }
};

// pass-3 twiddle W_n^{k r} for compile-time r = 4 a + b
template <int K3>
struct LTw3 {
  const float2* h;  // &TW3[0][k-1]
  float2 w1, w2, w3;
  template <int R_>
  __device__ __forceinline__ float2 at() const {
    constexpr int a = R_ >> 2, b = R_ & 3;
    const float2 t = h[a * K3];
    if constexpr (b == 0) return t;
    const float2 w = b == 1 ? w1 : (b == 2 ? w2 : w3);
    return make_float2(fmaf(t.x, w.x, -t.y * w.y), fmaf(t.x, w.y, t.y * w.x));
  }
};

// One closed set of a pass: window base `be`, block size m0, k in 1 .. m0/2 (k == m0/2: the
// zero-imaginary set), M blocks.  tw.template at<r>() = W_W^{k r} (forward) / conj (inverse).
template <typename P, int M, bool kInv, typename TW>
__device__ __forceinline__ void pl_set(float* H, int be, int m0, int k, const TW& tw) {
  constexpr int LM = ilog2c<M>();
  const int W = m0 * M;
  const bool half = (2 * k == m0);
  float zr[M], zi[M];
  if (!kInv) {
    ct::static_for<0, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      zr[j] = H[P::phys(be + j * m0 + k)];
      zi[j] = half ? 0.f : H[P::phys(be + (j + 1) * m0 - k)];
    });
    ct::static_for<1, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 t = tw.template at<rev_bits<LM>(j)>();
      const float q = zr[j];
      zr[j] = fmaf(q, t.x, -zi[j] * t.y);
      zi[j] = fmaf(q, t.y, zi[j] * t.x);
    });
    cfft_dit<M>(zr, zi);
    ct::static_for<0, M>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      if constexpr (q < M / 2) {
        H[P::phys(be + q * m0 + k)] = zr[q];
        H[P::phys(be + W - q * m0 - k)] = zi[q];
      } else {
        if (!half) {
          H[P::phys(be + q * m0 + k)] = -zi[q];
          H[P::phys(be + W - q * m0 - k)] = zr[q];
        }
      }
    });
  } else {
    // Y[q] into register rev(q): q < M/2: Re at q m0 + k, Im at W - q m0 - k;
    // q >= M/2: Re at W - q m0 - k, Im = -(value at q m0 + k)
    ct::static_for<0, M>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int rq = rev_bits<LM>(q);
      const float a = H[P::phys(be + q * m0 + k)], b = H[P::phys(be + W - q * m0 - k)];
      if constexpr (q < M / 2) {
        zr[rq] = a;
        zi[rq] = b;
      } else {
        zr[rq] = b;
        zi[rq] = -a;
      }
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
      H[P::phys(be + j * m0 + k)] = zr[rj];
      if (!half) H[P::phys(be + (j + 1) * m0 - k)] = zi[rj];
    });
  }
}

// DC set: slots be + j m0 (j < M) — the packed real M-point FFT (inverse: unscaled x scale).
template <typename P, int M, bool kInv>
__device__ __forceinline__ void pl_dc(float* H, int be, int m0, float scale) {
  float d[M];
  ct::static_for<0, M>([&](auto J) {
    constexpr int j = decltype(J)::value;
    d[j] = H[P::phys(be + j * m0)];
  });
  if (!kInv)
    rfft_fwd_reg<M>(d);
  else
    rfft_inv_reg<M>(d);
  ct::static_for<0, M>([&](auto J) {
    constexpr int j = decltype(J)::value;
    H[P::phys(be + j * m0)] = d[j] * scale;
  });
}

// pass-2 twiddle: TW2[j][k-1] = W_1024^{k rev5(j)} (conj for the inverse), indexed by natural j
struct LTw2 {
  const float2* h;  // &TW2[0][k-1]
  template <int R_>
  __device__ __forceinline__ float2 at() const {
    return h[rev_bits<5>(R_) * 16];
  }
};

template <typename T>
struct gio4;  // 4 consecutive elements <-> float4
template <>
struct gio4<float> {
  __device__ __forceinline__ static float4 ld(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
  __device__ __forceinline__ static void st(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }
};
template <>
struct gio4<__nv_bfloat16> {
  __device__ __forceinline__ static float4 ld(const __nv_bfloat16* p) {
    const uint2 u = __ldcs(reinterpret_cast<const uint2*>(p));
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u), __uint_as_float(u.y << 16),
                       __uint_as_float(u.y & 0xffff0000u));
  }
  __device__ __forceinline__ static void st(__nv_bfloat16* p, float4 v) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    __stcs(reinterpret_cast<uint2*>(p), make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b)));
  }
};

template <typename P, bool kInv>
__global__ void __launch_bounds__(P::NT, P::MINB) rdfftl_kernel(typename P::elem* __restrict__ x, int64_t batch) {
  using T = typename P::elem;
  constexpr int N = P::N, NT = P::NT, R = P::R, S = P::S, K3 = P::K3, M3 = P::M3;
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float* H = reinterpret_cast<float*>(base);
  float2* TW2 = reinterpret_cast<float2*>(base + P::TW2_OFF);
  float2* TW3 = reinterpret_cast<float2*>(base + P::TW3_OFF);
  const int tid = threadIdx.x;
  const float sg = kInv ? 1.0f : -1.0f;
  for (int e = tid; e < P::TW2N; e += NT) {
    const int j = e / 16, k = 1 + e % 16;
    float s, c;
    sincospif(2.0f * (float)(k * rev_bits<5>(j)) / 1024.0f, &s, &c);
    TW2[e] = make_float2(c, sg * s);
  }
  for (int e = tid; e < P::TW3N; e += NT) {
    const int a = e / K3, k = 1 + e % K3;
    float s, c;
    sincospif(2.0f * (float)(4 * k * a) / (float)N, &s, &c);
    TW3[e] = kInv ? make_float2(c * (1.0f / N), s * (1.0f / N)) : make_float2(c, -s);
  }
  // pass-3 sets k3 = tid + NT i (i < K3PT); k3 = 0 stands for the zero-imaginary set k3 = 512
  // plus the DC set (two real-input sets ~ one complex set of work)
  auto tw3_for = [&](int k3) {
    LTw3<K3> t;
    t.h = TW3 + (k3 - 1);
    float s, c;
    sincospif(2.0f * (float)k3 / (float)N, &s, &c);
    t.w1 = make_float2(c, sg * s);
    sincospif(4.0f * (float)k3 / (float)N, &s, &c);
    t.w2 = make_float2(c, sg * s);
    sincospif(6.0f * (float)k3 / (float)N, &s, &c);
    t.w3 = make_float2(c, sg * s);
    return t;
  };
  auto pass3 = [&](auto inv) {
    constexpr bool kI = decltype(inv)::value;
#pragma unroll 1
    for (int i = 0; i < P::K3PT; ++i) {
      const int kk = tid + NT * i, k3 = kk == 0 ? K3 : kk;
      pl_set<P, M3, kI>(H, 0, 1024, k3, tw3_for(k3));
      if (kk == 0) pl_dc<P, M3, kI>(H, 0, 1024, kI ? 1.0f / N : 1.0f);
    }
  };
  // pass-2 lane: window ww, k2 = 1 .. 15; lane 0 of each window: k2 = 16 (zero imaginary) + DC
  const int ww = tid / 16, k2 = tid % 16 == 0 ? 16 : tid % 16;
  const bool act2 = tid < P::NW2 * 16;
  LTw2 tw2;
  tw2.h = TW2 + (k2 - 1);
  const uint32_t k65536 = kTwo16;
  __syncthreads();
  for (int64_t v = blockIdx.x; v < batch; v += gridDim.x) {
    T* xv = x + v * (int64_t)N;
    if (!kInv) {
      if (tid < S / 2) {  // pass 1: subsequences 2c, 2c+1 -> windows rev(2c), rev(2c) + S/2
        const int c = tid;
        float2 b[R];
        ct::static_for<0, R>([&](auto I) {
          constexpr int i = decltype(I)::value;
          b[rev_bits<5>(i)] = gio<T>::ld2(xv + 2 * c + S * i, k65536);
        });
        rfft_fwd_reg<R>(b);
        const int w0 = rev_bits<P::LS>(2 * c), w1 = w0 + S / 2;
        ct::static_for<0, R / 4>([&](auto I) {
          constexpr int i = 4 * decltype(I)::value;
          *reinterpret_cast<float4*>(H + P::phys(w0 * 32 + i)) = make_float4(b[i].x, b[i + 1].x, b[i + 2].x, b[i + 3].x);
          *reinterpret_cast<float4*>(H + P::phys(w1 * 32 + i)) = make_float4(b[i].y, b[i + 1].y, b[i + 2].y, b[i + 3].y);
        });
      }
      __syncthreads();
      if (act2) pl_set<P, 32, false>(H, ww * 1024, 32, k2, tw2);
      if (act2 && k2 == 16) pl_dc<P, 32, false>(H, ww * 1024, 32, 1.0f);
      __syncthreads();
      pass3(std::false_type{});
      __syncthreads();
      for (int e = tid; e < N / 4; e += NT) {
        const float4 f = *reinterpret_cast<const float4*>(H + P::phys(4 * e));
        gio4<T>::st(xv + 4 * e, f);
      }
      __syncthreads();
    } else {
      for (int e = tid; e < N / 4; e += NT)
        *reinterpret_cast<float4*>(H + P::phys(4 * e)) = gio4<T>::ld(xv + 4 * e);
      __syncthreads();
      pass3(std::true_type{});
      __syncthreads();
      if (act2) pl_set<P, 32, true>(H, ww * 1024, 32, k2, tw2);
      if (act2 && k2 == 16) pl_dc<P, 32, true>(H, ww * 1024, 32, 1.0f);
      __syncthreads();
      if (tid < S / 2) {  // inverse pass 1
        const int c = tid;
        const int w0 = rev_bits<P::LS>(2 * c), w1 = w0 + S / 2;
        float2 b[R];
        ct::static_for<0, R / 4>([&](auto I) {
          constexpr int i = 4 * decltype(I)::value;
          const float4 f0 = *reinterpret_cast<const float4*>(H + P::phys(w0 * 32 + i));
          const float4 f1 = *reinterpret_cast<const float4*>(H + P::phys(w1 * 32 + i));
          b[i] = make_float2(f0.x, f1.x);
          b[i + 1] = make_float2(f0.y, f1.y);
          b[i + 2] = make_float2(f0.z, f1.z);
          b[i + 3] = make_float2(f0.w, f1.w);
        });
        rfft_inv_reg<R>(b);
        ct::static_for<0, R>([&](auto I) {
          constexpr int i = decltype(I)::value;
          gio<T>::st2(xv + 2 * c + S * i, b[rev_bits<5>(i)]);
        });
      }
      __syncthreads();
    }
  }
}

template <typename P>
bool launch_planl(typename P::elem* x, int64_t batch, bool inverse, int sms, cudaStream_t st) {
  auto kf = rdfftl_kernel<P, false>;
  auto ki = rdfftl_kernel<P, true>;
  static int per_sm = 0;
  if (!per_sm) {
    for (auto k : {kf, ki}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::BYTES);
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    }
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, kf, P::NT, P::BYTES);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ki, P::NT, P::BYTES);
    per_sm = a < b ? a : b;
    if (per_sm < 1) per_sm = 1;
    if (verbose())
      std::fprintf(stderr, "[rdfft] planL n=%d: %zu B smem, %d threads, %d CTAs/SM\n", P::N, (size_t)P::BYTES, P::NT,
                   per_sm);
  }
  const int grid = (int)(batch < (int64_t)per_sm * sms ? batch : (int64_t)per_sm * sms);
  if (inverse)
    ki<<<grid, P::NT, P::BYTES, st>>>(x, batch);
  else
    kf<<<grid, P::NT, P::BYTES, st>>>(x, batch);
  return true;
}

}  // namespace rdfft
