// bca_v1.cuh — fused block-circulant adapter (BCA) forward / backward.
//
// Forward (Eq. 4; blocks P:L184):  per token row t,
//   X_j = rdFFT(x_tj), Y_i = sum_j W_ij (.) X_j, y_ti = IrdFFT(Y_i),
// with W_ij = rdFFT(w_ij) computed once per CTA into shared memory (reading
// C12).  x is never modified (C13); every intermediate lives on chip, so the
// layer reads x and writes y exactly once.
//
// Backward (Eq. 5; blockwise pairing C11):  per token row t,
//   G_i = rdFFT(g_ti), X_j = rdFFT(x_tj)
//   dx_tj = IrdFFT(sum_i conj(W_ij) (.) G_i)          (dx may alias g: P:L432)
//   Acc_ij += conj(X_j) (.) G_i                         (per-CTA, fp32, smem)
// then Acc is added into dw with fp32 atomics and dw is inverse-transformed in
// place by the dw finalise launch (gradients in fp32).
#pragma once

#include "stages.cuh"

namespace rdfft {

constexpr int kBcaThreads = 512;

// Packed-domain (conj-)multiply-accumulate helpers over one bin k of length-p spectra.
// For k == 0 the real DC and Nyquist slots are handled together.
struct PackedBin {
  int p, k;
  __device__ __forceinline__ float2 get(const float* s) const {
    return k == 0 ? make_float2(s[0], s[p >> 1]) : make_float2(s[k], s[p - k]);
  }
  __device__ __forceinline__ void put(float* s, float2 v) const {
    if (k == 0) {
      s[0] = v.x;
      s[p >> 1] = v.y;
    } else {
      s[k] = v.x;
      s[p - k] = v.y;
    }
  }
  // DC/Nyquist are two independent real products; other bins are complex.
  __device__ __forceinline__ float2 mul(float2 a, float2 b) const {
    return k == 0 ? make_float2(a.x * b.x, a.y * b.y) : cmul(a, b);
  }
  __device__ __forceinline__ float2 mulc(float2 a, float2 b) const {  // a * conj(b)
    return k == 0 ? make_float2(a.x * b.x, a.y * b.y) : cmulc(a, b);
  }
};

__host__ __device__ constexpr size_t bca_fwd_smem_floats(int q_in, int q_out, int p) {
  return (size_t)p /*twiddles*/ + (size_t)q_out * q_in * p + (size_t)q_in * p + (size_t)q_out * p;
}
__host__ __device__ constexpr size_t bca_bwd_smem_floats(int q_in, int q_out, int p) {
  return (size_t)p + 2 * (size_t)q_out * q_in * p + (size_t)(q_in + q_out) * p + (size_t)q_in * p;
}

template <typename T>
__device__ __forceinline__ void bca_weight_spectra(const T* __restrict__ w, float* Wsp, int nblk, int p,
                                                   int logp, const float2* tw, const float* wspec) {
  if (wspec) {  // resident spectra (packed, natural order): a plain copy
    load_rows<float>(wspec, Wsp, nblk * p, p, logp, /*rev=*/false);
    __syncthreads();
    return;
  }
  load_rows<T>(w, Wsp, nblk * p, p, logp, /*rev=*/true);
  __syncthreads();
  fwd_stages_smem(Wsp, nblk, p, logp, tw);
}

template <typename T>
__global__ void __launch_bounds__(kBcaThreads) bca_fwd_v1_kernel(const T* __restrict__ x, const T* __restrict__ w,
                                                                   T* __restrict__ y, int64_t T_, int q_in,
                                                                   int q_out, int p, int logp, int yacc,
                                                                   const float* __restrict__ wspec) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  float2* tw = reinterpret_cast<float2*>(smem);
  float* Wsp = smem + p;
  float* Xs = Wsp + (size_t)q_out * q_in * p;
  float* Ys = Xs + (size_t)q_in * p;
  make_twiddles(tw, p);
  __syncthreads();
  bca_weight_spectra<T>(w, Wsp, q_out * q_in, p, logp, tw, wspec);
  const int hb = p >> 1;  // bins handled per block: k in [0, p/2)
  for (int64_t t = blockIdx.x; t < T_; t += gridDim.x) {
    load_rows<T>(x + t * q_in * p, Xs, q_in * p, p, logp, /*rev=*/true);
    __syncthreads();
    fwd_stages_smem(Xs, q_in, p, logp, tw);
    for (int it = threadIdx.x; it < q_out * hb; it += blockDim.x) {
      const int i = it / hb;
      const PackedBin bin{p, it - i * hb};
      float2 acc = make_float2(0.f, 0.f);
      for (int j = 0; j < q_in; ++j) {
        const float2 prod = bin.mul(bin.get(Wsp + ((size_t)i * q_in + j) * p), bin.get(Xs + (size_t)j * p));
        acc.x += prod.x;
        acc.y += prod.y;
      }
      bin.put(Ys + (size_t)i * p, acc);
    }
    __syncthreads();
    inv_stages_smem(Ys, q_out, p, logp, tw);
    store_rows<T>(y + t * q_out * p, Ys, q_out * p, p, logp, /*rev=*/true, yacc != 0);
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kBcaThreads) bca_bwd_v1_kernel(const T* __restrict__ x, const T* __restrict__ w,
                                                                   const T* g, T* dx, float* __restrict__ dw,
                                                                   int64_t T_, int q_in, int q_out, int p,
                                                                   int logp, const float* __restrict__ wspec) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  float2* tw = reinterpret_cast<float2*>(smem);
  const size_t nW = (size_t)q_out * q_in * p;
  float* Wsp = smem + p;
  float* Acc = Wsp + nW;
  float* XG = Acc + nW;                     // X_0..X_{q_in-1}, then G_0..G_{q_out-1}
  float* Gs = XG + (size_t)q_in * p;
  float* Ds = Gs + (size_t)q_out * p;
  make_twiddles(tw, p);
  for (size_t i = threadIdx.x; i < nW; i += blockDim.x) Acc[i] = 0.f;
  __syncthreads();
  bca_weight_spectra<T>(w, Wsp, q_out * q_in, p, logp, tw, wspec);
  const int hb = p >> 1;
  for (int64_t t = blockIdx.x; t < T_; t += gridDim.x) {
    load_rows<T>(x + t * q_in * p, XG, q_in * p, p, logp, /*rev=*/true);
    load_rows<T>(g + t * q_out * p, Gs, q_out * p, p, logp, /*rev=*/true);
    __syncthreads();
    fwd_stages_smem(XG, q_in + q_out, p, logp, tw);
    for (int it = threadIdx.x; it < q_in * hb; it += blockDim.x) {  // D_j = sum_i conj(W_ij) G_i
      const int j = it / hb;
      const PackedBin bin{p, it - j * hb};
      float2 acc = make_float2(0.f, 0.f);
      for (int i = 0; i < q_out; ++i) {
        const float2 prod = bin.mulc(bin.get(Gs + (size_t)i * p), bin.get(Wsp + ((size_t)i * q_in + j) * p));
        acc.x += prod.x;
        acc.y += prod.y;
      }
      bin.put(Ds + (size_t)j * p, acc);
    }
    for (int it = threadIdx.x; it < q_out * q_in * hb; it += blockDim.x) {  // Acc_ij += conj(X_j) G_i
      const int ij = it / hb;
      const int i = ij / q_in, j = ij - i * q_in;
      const PackedBin bin{p, it - ij * hb};
      const float2 prod = bin.mulc(bin.get(Gs + (size_t)i * p), bin.get(XG + (size_t)j * p));
      float* a = Acc + (size_t)ij * p;
      const float2 cur = bin.get(a);
      bin.put(a, make_float2(cur.x + prod.x, cur.y + prod.y));
    }
    __syncthreads();
    inv_stages_smem(Ds, q_in, p, logp, tw);
    store_rows<T>(dx + t * q_in * p, Ds, q_in * p, p, logp, /*rev=*/true);
    __syncthreads();
  }
  for (size_t i = threadIdx.x; i < nW; i += blockDim.x) atomicAdd(dw + i, Acc[i]);
}

}  // namespace rdfft
