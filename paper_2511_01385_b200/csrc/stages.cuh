// stages.cuh — block-cooperative in-place rdFFT stages on fp32 shared memory.
//
// The paper's schedule (§4.1 Prop. 1; §4.2 Eq. 7,
// P:L268-287), one __syncthreads per stage.  Used by the BCA kernels and the
// dw finalisation; the stand-alone transforms use the register-blocked
// kernels in rdfft_kernels.cuh.
//
// Forward stage merging packed m-blocks into packed 2m-blocks (block base b):
//   k = 0      : (b[0], b[m]) <- (b[0] + b[m], b[0] - b[m])             (both bins real)
//   k = m/2    : b[3m/2] <- -b[3m/2]                                   (Y_{m/2} = A - iB)
//   1<=k<m/2   : A = (b[k], b[m-k]), B = (b[m+k], b[2m-k]), u = W_{2m}^k B,
//                b[k] = Re(A+u), b[2m-k] = Im(A+u), b[m-k] = Re(A-u), b[m+k] = -Im(A-u)
// Inverse stage (reversed graph, reading C6): the exact inverse of the above with
// a factor 1/2 on the k = 0 pair and the general groups, none on k = m/2 (C4).
#pragma once

#include "common.cuh"

namespace rdfft {

// s: V vectors of length n (contiguous, fp32), already in bit-reversed order.
// tw: W_n^j table (j < n/2).  Ends with __syncthreads().
__device__ __forceinline__ void fwd_stages_smem(float* s, int V, int n, int logn, const float2* tw) {
  const int nt = blockDim.x;
  const int half = n >> 1;
  for (int idx = threadIdx.x; idx < V * half; idx += nt) {  // m = 1
    float* b = s + 2 * idx;
    const float a = b[0], c = b[1];
    b[0] = a + c;
    b[1] = a - c;
  }
  __syncthreads();
  const int quarter = n >> 2;
  for (int lm = 1; lm < logn; ++lm) {
    const int m = 1 << lm;
    const int hm = m >> 1;
    const int tws = logn - lm - 1;  // W_{2m}^k = W_n^{k n/(2m)}
    for (int idx = threadIdx.x; idx < V * quarter; idx += nt) {
      const int v = idx / quarter, r = idx - v * quarter;
      const int blk = r >> (lm - 1), k = r & (hm - 1);
      float* b = s + v * n + blk * 2 * m;
      if (k == 0) {
        const float a = b[0], c = b[m];
        b[0] = a + c;
        b[m] = a - c;
        b[m + hm] = -b[m + hm];
      } else {
        const float2 A = make_float2(b[k], b[m - k]);
        const float2 B = make_float2(b[m + k], b[2 * m - k]);
        const float2 u = cmul(tw[k << tws], B);
        b[k] = A.x + u.x;
        b[2 * m - k] = A.y + u.y;
        b[m - k] = A.x - u.x;
        b[m + k] = u.y - A.y;
      }
    }
    __syncthreads();
  }
}

// s: V packed spectra of length n.  Leaves bit-reversed real signals (the
// caller gathers with bitrev on the way out).  Ends with __syncthreads().
__device__ __forceinline__ void inv_stages_smem(float* s, int V, int n, int logn, const float2* tw) {
  const int nt = blockDim.x;
  const int quarter = n >> 2;
  for (int lm = logn - 1; lm >= 1; --lm) {
    const int m = 1 << lm;
    const int hm = m >> 1;
    const int tws = logn - lm - 1;
    for (int idx = threadIdx.x; idx < V * quarter; idx += nt) {
      const int v = idx / quarter, r = idx - v * quarter;
      const int blk = r >> (lm - 1), k = r & (hm - 1);
      float* b = s + v * n + blk * 2 * m;
      if (k == 0) {
        const float a = b[0], c = b[m];
        b[0] = 0.5f * (a + c);
        b[m] = 0.5f * (a - c);
        b[m + hm] = -b[m + hm];
      } else {
        const float2 Yk = make_float2(b[k], b[2 * m - k]);
        const float2 Ym = make_float2(b[m - k], -b[m + k]);  // Y_{m+k} = conj(Y_{m-k}) = A - u
        const float2 A = make_float2(0.5f * (Yk.x + Ym.x), 0.5f * (Yk.y + Ym.y));
        const float2 d = make_float2(0.5f * (Yk.x - Ym.x), 0.5f * (Yk.y - Ym.y));
        const float2 B = cmulc(d, tw[k << tws]);  // u / W = u conj(W)
        b[k] = A.x;
        b[m - k] = A.y;
        b[m + k] = B.x;
        b[2 * m - k] = B.y;
      }
    }
    __syncthreads();
  }
  const int half = n >> 1;
  for (int idx = threadIdx.x; idx < V * half; idx += nt) {  // m = 1
    float* b = s + 2 * idx;
    const float a = b[0], c = b[1];
    b[0] = 0.5f * (a + c);
    b[1] = 0.5f * (a - c);
  }
  __syncthreads();
}

// Load `count` elements (count = V*n) from global g into fp32 smem s, placing
// element i of each length-n row at its bit-reversed slot when `rev` is set.
template <typename T>
__device__ __forceinline__ void load_rows(const T* __restrict__ g, float* s, int count, int n, int logn,
                                          bool rev) {
  constexpr int VEC = io<T>::kVec;
  const int nvec = ((reinterpret_cast<uintptr_t>(g) & 15) == 0) ? count / VEC : 0;
  const uint4* g4 = reinterpret_cast<const uint4*>(g);
  for (int q = threadIdx.x; q < nvec; q += blockDim.x) {
    const uint4 u = __ldcs(g4 + q);
    float f[VEC];
    io<T>::unpack16(u, f);
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const int i = q * VEC + e;
      const int row = i >> logn, col = i & (n - 1);
      s[(row << logn) + (rev ? bitrev(col, logn) : col)] = f[e];
    }
  }
  for (int i = nvec * VEC + threadIdx.x; i < count; i += blockDim.x) {
    const int row = i >> logn, col = i & (n - 1);
    s[(row << logn) + (rev ? bitrev(col, logn) : col)] = io<T>::ld(g + i);
  }
}

// Store `count` elements to global g from fp32 smem s, reading element i of
// each row from its bit-reversed slot when `rev` is set; acc: g += values instead of g = values.
template <typename T>
__device__ __forceinline__ void store_rows(T* __restrict__ g, const float* s, int count, int n, int logn,
                                           bool rev, bool acc = false) {
  constexpr int VEC = io<T>::kVec;
  const int nvec = ((reinterpret_cast<uintptr_t>(g) & 15) == 0) ? count / VEC : 0;
  uint4* g4 = reinterpret_cast<uint4*>(g);
  for (int q = threadIdx.x; q < nvec; q += blockDim.x) {
    float f[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const int i = q * VEC + e;
      const int row = i >> logn, col = i & (n - 1);
      f[e] = s[(row << logn) + (rev ? bitrev(col, logn) : col)];
    }
    if (acc) {
      float o[VEC];
      io<T>::unpack16(g4[q], o);
#pragma unroll
      for (int e = 0; e < VEC; ++e) f[e] += o[e];
    }
    __stcs(g4 + q, io<T>::pack16(f));
  }
  for (int i = nvec * VEC + threadIdx.x; i < count; i += blockDim.x) {
    const int row = i >> logn, col = i & (n - 1);
    const float v = s[(row << logn) + (rev ? bitrev(col, logn) : col)];
    io<T>::st(g + i, acc ? v + io<T>::ld(g + i) : v);
  }
}

}  // namespace rdfft
