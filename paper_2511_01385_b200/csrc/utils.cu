// utils.cu — packed-spectrum utilities: decode / encode between the packed
// layout and the interleaved rFFT layout, conjugation and axpy in the packed
// domain.  Memory-bound elementwise kernels: each element is read once and written once with
// 16-byte (conj, axpy) or pair (decode, encode) accesses; grid-stride persistent grids.
//
//  * decode (the "decode step" of the Limitations): packed row p[n] ->
//    c[n + 2] = (Re y_0, Im y_0, ..., Re y_{n/2}, Im y_{n/2}) with Im y_0 = Im y_{n/2} = 0.
//  * encode: the inverse map (Im y_0, Im y_{n/2} are ignored: zero for a Hermitian spectrum).
//  * conj:  y_k -> conj(y_k) is a sign flip of slots n/2 + 1 .. n - 1 (a bit operation, exact).
//  * axpy:  y <- y + alpha x; the packing is linear, so this is the spectral-domain axpy
//    (and, with alpha = -lr, a spectral-domain SGD step).
#include "common.cuh"
#include "fast.h"

namespace rdfft {

namespace {

constexpr int kUThreads = 256;

template <typename T>
struct vec16;  // 16-byte vector of T as raw words
template <>
struct vec16<float> {
  static constexpr int E = 4;
};
template <>
struct vec16<__nv_bfloat16> {
  static constexpr int E = 8;
};

// sign-flip mask of element `col` (bits of one T)
template <typename T>
__device__ __forceinline__ uint32_t neg_bit(int col, int n) {
  return col > n / 2 ? (sizeof(T) == 4 ? 0x80000000u : 0x8000u) : 0u;
}

template <typename T>
__global__ void __launch_bounds__(kUThreads) packed_conj_kernel(T* __restrict__ a, int64_t total, int n, int logn) {
  constexpr int E = vec16<T>::E;
  const int64_t nvec = total / E;
  uint4* a4 = reinterpret_cast<uint4*>(a);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = v * E;  // a vector may span several rows when n < E
    uint4 u = __ldcs(a4 + v);
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
    if (n >= 2 * E) {
      // the 16-byte vector holds E consecutive columns c0 .. c0 + E - 1 of one row, and n/2 is a multiple
      // of E: every column flips (c0 > n/2), none does (c0 < n/2), or all but the first (c0 == n/2)
      const int c0 = (int)(e0 & (n - 1));
      const uint32_t m = c0 >= n / 2 ? (sizeof(T) == 4 ? 0x80000000u : 0x80008000u) : 0u;
      w[0] ^= (c0 == n / 2) ? (sizeof(T) == 4 ? 0u : 0x80000000u) : m;
      w[1] ^= m;
      w[2] ^= m;
      w[3] ^= m;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if constexpr (sizeof(T) == 4) {
          w[i] ^= neg_bit<T>((int)((e0 + i) & (n - 1)), n);
        } else {
          w[i] ^= neg_bit<T>((int)((e0 + 2 * i) & (n - 1)), n) |
                  (neg_bit<T>((int)((e0 + 2 * i + 1) & (n - 1)), n) << 16);
        }
      }
    }
    __stcs(a4 + v, make_uint4(w[0], w[1], w[2], w[3]));
  }
  // ragged tail (total % E elements; only when n < E, i.e. tiny rows)
  for (int64_t e = nvec * E + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(e & (n - 1));
    if (col > n / 2) {
      if constexpr (sizeof(T) == 4)
        a[e] = -a[e];
      else
        a[e] = __hneg(a[e]);
    }
  }
  (void)logn;
}

template <typename T>
__device__ __forceinline__ void unpack_words(uint4 u, float* f) {
  if constexpr (sizeof(T) == 4) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  } else {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
}
template <typename T>
__device__ __forceinline__ uint4 pack_words(const float* f) {
  if constexpr (sizeof(T) == 4) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  } else {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);  // RNE (reading C7)
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// y <- y + alpha x (x broadcast when x_rows == 1: row length n)
template <typename T>
__global__ void __launch_bounds__(kUThreads) packed_axpy_kernel(T* __restrict__ y, const T* __restrict__ x,
                                                               float alpha, int64_t total, int n, bool bcast,
                                                               bool vec) {
  constexpr int E = vec16<T>::E;
  const int64_t nvec = vec ? total / E : 0;
  uint4* y4 = reinterpret_cast<uint4*>(y);
  const uint4* x4 = reinterpret_cast<const uint4*>(x);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t xv = bcast ? (v & ((n / E) - 1)) : v;
    float fy[E], fx[E];
    unpack_words<T>(__ldcs(y4 + v), fy);
    unpack_words<T>(bcast ? __ldg(x4 + xv) : __ldcs(x4 + xv), fx);
#pragma unroll
    for (int i = 0; i < E; ++i) fy[i] = fmaf(alpha, fx[i], fy[i]);
    __stcs(y4 + v, pack_words<T>(fy));
  }
  for (int64_t e = nvec * E + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t xe = bcast ? (e & (n - 1)) : e;
    y[e] = (T)fmaf(alpha, (float)x[xe], (float)y[e]);
  }
}

// element pair (v0, v1) store / load of T
template <typename T>
__device__ __forceinline__ void st_pair(T* p, T v0, T v1) {
  if constexpr (sizeof(T) == 4) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v0, v1));
  } else {
    __nv_bfloat162 h;
    h.x = v0;
    h.y = v1;
    __stcs(reinterpret_cast<unsigned int*>(p), *reinterpret_cast<unsigned int*>(&h));
  }
}
template <typename T>
__device__ __forceinline__ void ld_pair(const T* p, T& v0, T& v1) {
  if constexpr (sizeof(T) == 4) {
    const float2 f = __ldcs(reinterpret_cast<const float2*>(p));
    v0 = f.x;
    v1 = f.y;
  } else {
    const unsigned int u = __ldcs(reinterpret_cast<const unsigned int*>(p));
    const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&u);
    v0 = h.x;
    v1 = h.y;
  }
}

// decode / encode stage the packed rows of a CTA's row chunk in shared memory: the packed side moves
// with coalesced 16-byte accesses, and the mirrored slot n - k of a bin is read / written in shared
// memory instead of HBM; the interleaved side moves one bin pair (4 / 8 bytes) per thread, consecutive
// bins on consecutive lanes.  (One bin per thread straight from HBM with 2-byte mirrored accesses ran
// at 0.28-0.52 of HBM.)  Rows of at least 16 bytes (n * sizeof(T) % 16 == 0), rows_per_cta * n <= kUSm.
constexpr int kU = 4;
constexpr int kUSm = 4096;  // elements of the staged chunk (8 / 16 KB)
// e / nb for 0 <= e < 2^22 without an integer division: a float-reciprocal estimate and one
// correction step (the estimate is within one of the true quotient at these magnitudes)
__device__ __forceinline__ int div_nb(int e, int nb, float inv_nb) {
  int q = __float2int_rz((float)e * inv_nb);
  const int r = e - q * nb;
  q += (r >= nb) - (r < 0);
  return q;
}

template <typename T>
__global__ void __launch_bounds__(kUThreads) decode_staged_kernel(const T* __restrict__ p, T* __restrict__ c,
                                                                 int64_t batch, int n, int rows_per_cta) {
  __shared__ uint4 sm4[kUSm * sizeof(T) / 16];
  const T* sm = reinterpret_cast<const T*>(sm4);
  const int nb = n / 2 + 1;
  const T zero = T(0.0f);
  const float inv_nb = 1.0f / (float)nb;
  constexpr int E = 16 / (int)sizeof(T);
  for (int64_t r0 = (int64_t)blockIdx.x * rows_per_cta; r0 < batch; r0 += (int64_t)gridDim.x * rows_per_cta) {
    const int rows = (int)(batch - r0 < rows_per_cta ? batch - r0 : rows_per_cta);
    const uint4* src = reinterpret_cast<const uint4*>(p + r0 * n);
    __syncthreads();  // the previous chunk's reads of sm are done
    for (int i = threadIdx.x; i < rows * n / E; i += kUThreads) sm4[i] = __ldcs(src + i);
    for (int i = rows * n / E * E + threadIdx.x; i < rows * n; i += kUThreads)  // n < E: ragged chunk
      const_cast<T*>(sm)[i] = p[r0 * n + i];
    __syncthreads();
    const int tot = rows * nb;
    for (int e0 = threadIdx.x; e0 < tot; e0 += kU * kUThreads) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kUThreads;
        if (e < tot) {
          const int rr = div_nb(e, nb, inv_nb), k = e - rr * nb;
          const T* pr = sm + rr * n;
          const T im = (k == 0 || k == n / 2) ? zero : pr[n - k];
          st_pair<T>(c + (r0 + rr) * (int64_t)(n + 2) + 2 * k, pr[k], im);
        }
      }
    }
  }
}

// interleaved bins [batch][n + 2] -> packed rows [batch][n] (the mirror of decode_kernel)
template <typename T>
__global__ void __launch_bounds__(kUThreads) encode_staged_kernel(const T* __restrict__ c, T* __restrict__ p,
                                                                 int64_t batch, int n, int rows_per_cta) {
  __shared__ uint4 sm4[kUSm * sizeof(T) / 16];
  T* sm = reinterpret_cast<T*>(sm4);
  const int nb = n / 2 + 1;
  const float inv_nb = 1.0f / (float)nb;
  constexpr int E = 16 / (int)sizeof(T);
  for (int64_t r0 = (int64_t)blockIdx.x * rows_per_cta; r0 < batch; r0 += (int64_t)gridDim.x * rows_per_cta) {
    const int rows = (int)(batch - r0 < rows_per_cta ? batch - r0 : rows_per_cta);
    const int tot = rows * nb;
    __syncthreads();  // the previous chunk's stores from sm are done
    for (int e0 = threadIdx.x; e0 < tot; e0 += kU * kUThreads) {
      T re[kU], im[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kUThreads;
        if (e < tot) {
          const int rr = div_nb(e, nb, inv_nb), k = e - rr * nb;
          ld_pair<T>(c + (r0 + rr) * (int64_t)(n + 2) + 2 * k, re[u], im[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kUThreads;
        if (e < tot) {
          const int rr = div_nb(e, nb, inv_nb), k = e - rr * nb;
          T* pr = sm + rr * n;
          pr[k] = re[u];
          if (k != 0 && k != n / 2) pr[n - k] = im[u];
        }
      }
    }
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(p + r0 * n);
    for (int i = threadIdx.x; i < rows * n / E; i += kUThreads) __stcs(dst + i, sm4[i]);
    for (int i = rows * n / E * E + threadIdx.x; i < rows * n; i += kUThreads) p[r0 * n + i] = sm[i];  // n < E
  }
}

// n > kUSm (one row does not fit the staged chunk): one bin per thread straight from HBM
template <typename T>
__global__ void __launch_bounds__(kUThreads) decode_direct_kernel(const T* __restrict__ p, T* __restrict__ c,
                                                                 int64_t batch, int n) {
  const int nb = n / 2 + 1;
  const T zero = T(0.0f);
  for (int64_t r = blockIdx.x; r < batch; r += gridDim.x) {
    const T* pr = p + r * n;
    for (int k = threadIdx.x; k < nb; k += kUThreads) {
      const T im = (k == 0 || k == n / 2) ? zero : pr[n - k];
      st_pair<T>(c + r * (int64_t)(n + 2) + 2 * k, pr[k], im);
    }
  }
}
template <typename T>
__global__ void __launch_bounds__(kUThreads) encode_direct_kernel(const T* __restrict__ c, T* __restrict__ p,
                                                                 int64_t batch, int n) {
  const int nb = n / 2 + 1;
  for (int64_t r = blockIdx.x; r < batch; r += gridDim.x) {
    T* pr = p + r * n;
    for (int k = threadIdx.x; k < nb; k += kUThreads) {
      T re, im;
      ld_pair<T>(c + r * (int64_t)(n + 2) + 2 * k, re, im);
      pr[k] = re;
      if (k != 0 && k != n / 2) pr[n - k] = im;
    }
  }
}

// a <- a (.) [conj] b per bin for rows longer than the tiled kernel's 16 KB tiles (n > 4096):
// bins k = 0 .. n/2 of a row, (slot k, slot n - k) pairs; kU bins per thread per step with
// all loads issued before the first store (decode_kernel's schedule).
template <typename T, bool kConj>
__global__ void __launch_bounds__(kUThreads) packed_mul_large_kernel(T* __restrict__ a, const T* __restrict__ b,
                                                                    int64_t batch, int n, bool bcast) {
  const int nb = n / 2 + 1;
  const int64_t total = batch * nb;
  const int64_t step = (int64_t)gridDim.x * kUThreads;
  const double inv_nb = 1.0 / (double)nb;
  for (int64_t e0 = blockIdx.x * (int64_t)kUThreads + threadIdx.x; e0 < total; e0 += kU * step) {
    float xr[kU], xi[kU], yr[kU], yi[kU];
    T* ar[kU];
    int kk[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t e = e0 + u * step;
      ar[u] = nullptr;
      if (e < total) {
        int64_t r = (int64_t)((double)e * inv_nb);  // e / nb: fp64 reciprocal + one correction (e < 2^50)
        int k = (int)(e - r * nb);
        if (k >= nb) { ++r; k -= nb; }
        if (k < 0) { --r; k += nb; }
        ar[u] = a + r * n;
        kk[u] = k;
        const T* br = b + (bcast ? 0 : r * n);
        const bool real = (k == 0 || k == n / 2);
        xr[u] = (float)ar[u][k];
        yr[u] = (float)br[k];
        xi[u] = real ? 0.f : (float)ar[u][n - k];
        yi[u] = real ? 0.f : (kConj ? -(float)br[n - k] : (float)br[n - k]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (ar[u] != nullptr) {
        const int k = kk[u];
        if (k == 0 || k == n / 2) {  // real bins
          ar[u][k] = (T)(xr[u] * yr[u]);
        } else {
          ar[u][k] = (T)fmaf(xr[u], yr[u], -xi[u] * yi[u]);
          ar[u][n - k] = (T)fmaf(xr[u], yi[u], xi[u] * yr[u]);
        }
      }
    }
  }
}

int grid_of(int64_t work_items, int sms) {
  const int64_t blocks = (work_items + kUThreads - 1) / kUThreads;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(blocks < 1 ? 1 : (blocks < cap ? blocks : cap));
}

}  // namespace

template <typename T>
void launch_packed_conj(T* a, int64_t batch, int n, int logn, int sms, cudaStream_t st) {
  const int64_t total = batch * (int64_t)n;
  packed_conj_kernel<T><<<grid_of(total / vec16<T>::E + 1, sms), kUThreads, 0, st>>>(a, total, n, logn);
}
template <typename T>
void launch_packed_axpy(T* y, const T* x, float alpha, int64_t batch, int n, bool bcast, int sms, cudaStream_t st) {
  const int64_t total = batch * (int64_t)n;
  // broadcast needs whole 16-byte vectors per row: n >= E (else the scalar tail loop does it all)
  const bool vec = !bcast || n >= vec16<T>::E;  // tiny broadcast rows: scalar loop only
  packed_axpy_kernel<T><<<grid_of(vec ? total / vec16<T>::E + 1 : total, sms), kUThreads, 0, st>>>(
      y, x, alpha, total, n, bcast, vec);
}
template <typename T>
void launch_decode(const T* p, T* c, int64_t batch, int n, int sms, cudaStream_t st) {
  if (n > kUSm) {
    const int grid = (int)(batch < (int64_t)sms * 8 ? batch : (int64_t)sms * 8);
    decode_direct_kernel<T><<<grid, kUThreads, 0, st>>>(p, c, batch, n);
    return;
  }
  const int rows = kUSm / n;
  const int64_t ctas = (batch + rows - 1) / rows;
  const int grid = (int)(ctas < (int64_t)sms * 8 ? ctas : (int64_t)sms * 8);
  decode_staged_kernel<T><<<grid, kUThreads, 0, st>>>(p, c, batch, n, rows);
}
template <typename T>
void launch_encode(const T* c, T* p, int64_t batch, int n, int sms, cudaStream_t st) {
  if (n > kUSm) {
    const int grid = (int)(batch < (int64_t)sms * 8 ? batch : (int64_t)sms * 8);
    encode_direct_kernel<T><<<grid, kUThreads, 0, st>>>(c, p, batch, n);
    return;
  }
  const int rows = kUSm / n;
  const int64_t ctas = (batch + rows - 1) / rows;
  const int grid = (int)(ctas < (int64_t)sms * 8 ? ctas : (int64_t)sms * 8);
  encode_staged_kernel<T><<<grid, kUThreads, 0, st>>>(c, p, batch, n, rows);
}

template <typename T>
void launch_packed_mul_large(T* a, const T* b, int64_t batch, int n, bool bcast, bool conj, int sms, cudaStream_t st) {
  const int grid = grid_of(batch * (n / 2 + 1), sms);
  if (conj)
    packed_mul_large_kernel<T, true><<<grid, kUThreads, 0, st>>>(a, b, batch, n, bcast);
  else
    packed_mul_large_kernel<T, false><<<grid, kUThreads, 0, st>>>(a, b, batch, n, bcast);
}

#define RDFFT_UTILS_INST(T)                                                                                   \
  template void launch_packed_conj<T>(T*, int64_t, int, int, int, cudaStream_t);                              \
  template void launch_packed_axpy<T>(T*, const T*, float, int64_t, int, bool, int, cudaStream_t);             \
  template void launch_decode<T>(const T*, T*, int64_t, int, int, cudaStream_t);                               \
  template void launch_encode<T>(const T*, T*, int64_t, int, int, cudaStream_t);                               \
  template void launch_packed_mul_large<T>(T*, const T*, int64_t, int, bool, bool, int, cudaStream_t);
RDFFT_UTILS_INST(float)
RDFFT_UTILS_INST(__nv_bfloat16)
#undef RDFFT_UTILS_INST

}  // namespace rdfft
