// abi.cu — the C-ABI of librdfft.so (declared and documented in include/rdfft.h).
//
// Host side only: validate arguments, pick a kernel configuration from
// (n, dtype) alone (never from batch, so any sharding of the batch gives
// bit-identical rows), launch on the caller's stream.  No allocation.
#include <atomic>
#include <cstdio>
#include <cstring>

#include "../../include/rdfft.h"
#include "bca_v1.cuh"
#include "bca_tiled.cuh"
#include "kernels_v1.cuh"
#include "fast.h"

using namespace rdfft;

namespace {

std::atomic<uint64_t> g_launches{0};

int ilog2(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}
// BCA blocks: 2 <= p <= 4096 (reading C9); transforms, packed products and the utilities also
// take the large sizes of SURVEY §8(f) N2, n <= 65536 (planl.cuh; 65536 on cluster pairs).
constexpr int64_t kMaxTransformN = 65536;
bool pow2_in_range(int64_t n) { return n >= 2 && n <= kMaxN && (n & (n - 1)) == 0; }
bool pow2_transform(int64_t n) { return n >= 2 && n <= kMaxTransformN && (n & (n - 1)) == 0; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* pa = static_cast<const char*>(a);
  const char* pb = static_cast<const char*>(b);
  return na && nb && pa < pb + nb && pb < pa + na;
}
size_t dsize(int dtype) { return dtype == RDFFT_BF16 ? 2 : 4; }

int num_sms() {  // per device (a process may drive several GPUs)
  static int sms_dev[kMaxDevices] = {};
  const int dev = device_index();
  int& sms = sms_dev[dev];
  if (!sms) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int launched(int count = 1) {
  g_launches.fetch_add(count, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? RDFFT_OK : RDFFT_E_CUDA;
}

// Every legal n has a specialised kernel (plan3.cuh dispatch); a launcher that could not launch
// (e.g. cudaLaunchKernelEx of the n = 65536 cluster pair failed) is reported, never replaced.
template <typename T>
int launch_transform(T* x, int64_t batch, int n, bool inverse, cudaStream_t st) {
  if (launch_rdfft_fast<T>(x, batch, n, ilog2(n), inverse, num_sms(), st)) return launched();
  (void)cudaGetLastError();
  return RDFFT_E_CUDA;
}

int transform(void* x, int64_t batch, int64_t n, int dtype, void* stream, bool inverse) {
  if (dtype != RDFFT_F32 && dtype != RDFFT_BF16) return RDFFT_E_DTYPE;
  if (!pow2_transform(n)) return RDFFT_E_SIZE;
  if (batch < 0) return RDFFT_E_SHAPE;
  if (batch == 0) return RDFFT_OK;
  if (!x) return RDFFT_E_NULL;
  if (!aligned16(x)) return RDFFT_E_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == RDFFT_F32) return launch_transform<float>(static_cast<float*>(x), batch, (int)n, inverse, st);
  return launch_transform<__nv_bfloat16>(static_cast<__nv_bfloat16*>(x), batch, (int)n, inverse, st);
}

int packed(void* a, const void* b, int64_t batch, int64_t n, int64_t b_batch, int dtype, void* stream, bool conj) {
  if (dtype != RDFFT_F32 && dtype != RDFFT_BF16) return RDFFT_E_DTYPE;
  if (!pow2_transform(n)) return RDFFT_E_SIZE;
  if (batch < 0 || b_batch < 0) return RDFFT_E_SHAPE;
  if (batch == 0) return RDFFT_OK;
  if (b_batch != 1 && b_batch != batch) return RDFFT_E_SHAPE;
  if (!a || !b) return RDFFT_E_NULL;
  if (!aligned16(a) || !aligned16(b)) return RDFFT_E_ALIGN;
  const size_t s = dsize(dtype);
  if (overlap(a, batch * n * s, b, b_batch * n * s) && !(a == b && b_batch == batch)) return RDFFT_E_ALIAS;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int logn = ilog2(n);
  if (n > kMaxN) {  // rows longer than the tiled kernels' tiles
    if (dtype == RDFFT_F32)
      launch_packed_mul_large<float>(static_cast<float*>(a), static_cast<const float*>(b), batch, (int)n,
                                     b_batch == 1 && batch > 1, conj, num_sms(), st);
    else
      launch_packed_mul_large<__nv_bfloat16>(static_cast<__nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(b),
                                             batch, (int)n, b_batch == 1 && batch > 1, conj, num_sms(), st);
    return launched();
  }
  if (n >= 16 && aligned16(a) && aligned16(b)) {
    const int rows = (kPm2TileBytes / (int)s) >> logn;
    const int64_t tiles = (batch + rows - 1) / rows;
    const size_t smem = (size_t)kPm2Stages * kPm2TileBytes +
                        (b_batch == 1 ? ((n * s + 15) & ~(size_t)15) : (size_t)kPm2Stages * kPm2TileBytes) +
                        (2 * kPm2Stages + 1) * 8;
    if (dtype == RDFFT_F32) {
      for (auto k : {packed_mul2_kernel<float, false>, packed_mul2_kernel<float, true>})
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
    } else {
      for (auto k : {packed_mul2_kernel<__nv_bfloat16, false>, packed_mul2_kernel<__nv_bfloat16, true>})
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
    }
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / (smem + 1024)));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * per_sm));
#define RDFFT_PM2(T, C) \
  packed_mul2_kernel<T, C><<<grid, kPm2Threads, smem, st>>>(static_cast<T*>(a), static_cast<const T*>(b), batch, (int)n, logn, b_batch)
    if (dtype == RDFFT_F32) {
      if (conj) RDFFT_PM2(float, true); else RDFFT_PM2(float, false);
    } else {
      if (conj) RDFFT_PM2(__nv_bfloat16, true); else RDFFT_PM2(__nv_bfloat16, false);
    }
#undef RDFFT_PM2
    return launched();
  }
  const int rows = (kPmTileBytes / (int)s) >> logn;
  const int64_t tiles = (batch + rows - 1) / rows;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * 6));
#define RDFFT_PM(T, C) \
  packed_mul_kernel<T, C><<<grid, kPmThreads, 0, st>>>(static_cast<T*>(a), static_cast<const T*>(b), batch, (int)n, logn, b_batch)
  if (dtype == RDFFT_F32) {
    if (conj) RDFFT_PM(float, true); else RDFFT_PM(float, false);
  } else {
    if (conj) RDFFT_PM(__nv_bfloat16, true); else RDFFT_PM(__nv_bfloat16, false);
  }
#undef RDFFT_PM
  return launched();
}

int bca_check(const void* x, const void* w, int64_t T, int64_t d_in, int64_t d_out, int64_t p, int dtype) {
  if (dtype != RDFFT_F32 && dtype != RDFFT_BF16) return RDFFT_E_DTYPE;
  if (!pow2_in_range(p)) return RDFFT_E_SIZE;
  if (T < 0 || d_in <= 0 || d_out <= 0 || d_in % p || d_out % p) return RDFFT_E_SHAPE;
  if (!x || !w) return T == 0 ? RDFFT_OK : RDFFT_E_NULL;
  if (!aligned16(x) || !aligned16(w)) return RDFFT_E_ALIGN;
  return RDFFT_OK;
}

template <typename K>
int grid_for(K kernel, int threads, size_t smem, int64_t units) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm <= 0) return 0;
  return (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)per_sm * num_sms()));
}


int bca_fwd_tiled(const void* x, const void* w, void* y, int64_t T, int q_in, int q_out, int p, int logp, int dtype,
                  cudaStream_t st, int acc, const float* wspec) {
  BcaTiledPlan plan{};
  if (!bca_tiled_plan(false, false, T, q_in, q_out, p, num_sms(), &plan)) return RDFFT_E_SHAPE;
  const dim3 grid((unsigned)std::min<int64_t>(plan.tiles, (int64_t)num_sms() * 4), (unsigned)plan.groups);
  if (dtype == RDFFT_F32) {
    auto k = bca_fwd_tiled_kernel<float>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
    k<<<grid, kBcaTiledThreads, plan.smem, st>>>(static_cast<const float*>(x), static_cast<const float*>(w),
                                                  static_cast<float*>(y), T, q_in, q_out, p, logp, plan.vt, plan.grp,
                                                  acc, wspec);
  } else {
    auto k = bca_fwd_tiled_kernel<__nv_bfloat16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
    k<<<grid, kBcaTiledThreads, plan.smem, st>>>(static_cast<const __nv_bfloat16*>(x),
                                                  static_cast<const __nv_bfloat16*>(w),
                                                  static_cast<__nv_bfloat16*>(y), T, q_in, q_out, p, logp, plan.vt,
                                                  plan.grp, acc, wspec);
  }
  return launched();
}

// shared validation of the packed-spectrum utilities: 1 = proceed, 0 = no-op, < 0 = -status
int util_check(const void* a, const void* b, int64_t batch, int64_t n, int dtype) {
  if (dtype != RDFFT_F32 && dtype != RDFFT_BF16) return -RDFFT_E_DTYPE;
  if (!pow2_transform(n)) return -RDFFT_E_SIZE;
  if (batch < 0) return -RDFFT_E_SHAPE;
  if (batch == 0) return 0;
  if (!a || !b) return -RDFFT_E_NULL;
  if (!aligned16(a) || !aligned16(b)) return -RDFFT_E_ALIGN;
  return 1;
}

}  // namespace

extern "C" {

int rdfft_decode(const void* p, void* c, int64_t batch, int64_t n, int dtype, void* stream) {
  const int ok = util_check(p, c, batch, n, dtype);
  if (ok <= 0) return -ok;
  const size_t s = dsize(dtype);
  if (overlap(p, batch * n * s, c, batch * (n + 2) * s)) return RDFFT_E_ALIAS;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == RDFFT_F32)
    launch_decode<float>(static_cast<const float*>(p), static_cast<float*>(c), batch, (int)n, num_sms(), st);
  else
    launch_decode<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(p), static_cast<__nv_bfloat16*>(c), batch,
                                 (int)n, num_sms(), st);
  return launched();
}

int rdfft_encode(const void* c, void* p, int64_t batch, int64_t n, int dtype, void* stream) {
  const int ok = util_check(c, p, batch, n, dtype);
  if (ok <= 0) return -ok;
  const size_t s = dsize(dtype);
  if (overlap(p, batch * n * s, c, batch * (n + 2) * s)) return RDFFT_E_ALIAS;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == RDFFT_F32)
    launch_encode<float>(static_cast<const float*>(c), static_cast<float*>(p), batch, (int)n, num_sms(), st);
  else
    launch_encode<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(c), static_cast<__nv_bfloat16*>(p), batch,
                                 (int)n, num_sms(), st);
  return launched();
}

int rdfft_packed_conj(void* a, int64_t batch, int64_t n, int dtype, void* stream) {
  const int ok = util_check(a, a, batch, n, dtype);
  if (ok <= 0) return -ok;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == RDFFT_F32)
    launch_packed_conj<float>(static_cast<float*>(a), batch, (int)n, ilog2(n), num_sms(), st);
  else
    launch_packed_conj<__nv_bfloat16>(static_cast<__nv_bfloat16*>(a), batch, (int)n, ilog2(n), num_sms(), st);
  return launched();
}

int rdfft_packed_axpy(void* y, const void* x, float alpha, int64_t batch, int64_t n, int64_t x_batch, int dtype,
                      void* stream) {
  const int ok = util_check(y, x, batch, n, dtype);
  if (ok < 0) return -ok;
  if (x_batch < 0 || (batch > 0 && x_batch != 1 && x_batch != batch)) return RDFFT_E_SHAPE;
  if (ok == 0) return RDFFT_OK;
  const size_t s = dsize(dtype);
  if (overlap(y, batch * n * s, x, x_batch * n * s) && !(y == x && x_batch == batch)) return RDFFT_E_ALIAS;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool bcast = x_batch == 1 && batch > 1;
  if (dtype == RDFFT_F32)
    launch_packed_axpy<float>(static_cast<float*>(y), static_cast<const float*>(x), alpha, batch, (int)n, bcast,
                              num_sms(), st);
  else
    launch_packed_axpy<__nv_bfloat16>(static_cast<__nv_bfloat16*>(y), static_cast<const __nv_bfloat16*>(x), alpha,
                                      batch, (int)n, bcast, num_sms(), st);
  return launched();
}

int rdfft_fwd(void* x, int64_t batch, int64_t n, int dtype, void* stream) {
  return transform(x, batch, n, dtype, stream, false);
}

int rdfft_inv(void* x, int64_t batch, int64_t n, int dtype, void* stream) {
  return transform(x, batch, n, dtype, stream, true);
}

int rdfft_packed_mul(void* a, const void* b, int64_t batch, int64_t n, int64_t b_batch, int dtype, void* stream) {
  return packed(a, b, batch, n, b_batch, dtype, stream, false);
}

int rdfft_packed_conjmul(void* a, const void* b, int64_t batch, int64_t n, int64_t b_batch, int dtype,
                         void* stream) {
  return packed(a, b, batch, n, b_batch, dtype, stream, true);
}

// wspec: the caller's resident weight spectra (fp32 packed, [q_out][q_in][p]) instead of w
static int bca_fwd_impl(const void* x, const void* w, void* y, int64_t T, int64_t d_in, int64_t d_out, int64_t p,
                        int dtype, void* stream, int acc, const float* wspec = nullptr) {
  if (wspec) w = wspec;  // validated and alias-checked as the weight operand (fp32: see ws below)
  int rc = bca_check(x, w, T, d_in, d_out, p, dtype);
  if (rc != RDFFT_OK || T == 0) return rc;
  if (!y) return RDFFT_E_NULL;
  if (!aligned16(y)) return RDFFT_E_ALIGN;
  const size_t s = dsize(dtype);
  const int q_in = (int)(d_in / p), q_out = (int)(d_out / p);
  const size_t ws = wspec ? 4 : s;
  if (overlap(y, T * d_out * s, x, T * d_in * s) || overlap(y, T * d_out * s, w, (size_t)q_out * q_in * p * ws))
    return RDFFT_E_ALIAS;
  const size_t smem = bca_fwd_smem_floats(q_in, q_out, (int)p) * sizeof(float);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int logp = ilog2(p);
  if (smem > 227 * 1024) return bca_fwd_tiled(x, w, y, T, q_in, q_out, (int)p, logp, dtype, st, acc, wspec);
  const bool fast =
      dtype == RDFFT_F32
          ? bca_fwd_fast<float>(static_cast<const float*>(x), static_cast<const float*>(w), static_cast<float*>(y), T,
                                q_in, q_out, (int)p, num_sms(), st, acc, wspec)
          : bca_fwd_fast<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
                                        static_cast<__nv_bfloat16*>(y), T, q_in, q_out, (int)p, num_sms(), st, acc,
                                        wspec);
  if (fast) return launched();
  if (dtype == RDFFT_F32) {
    auto k = bca_fwd_v1_kernel<float>;
    const int grid = grid_for(k, kBcaThreads, smem, T);
    if (!grid) return RDFFT_E_SHAPE;
    k<<<grid, kBcaThreads, smem, st>>>(static_cast<const float*>(x), static_cast<const float*>(w),
                                       static_cast<float*>(y), T, q_in, q_out, (int)p, logp, acc, wspec);
  } else {
    auto k = bca_fwd_v1_kernel<__nv_bfloat16>;
    const int grid = grid_for(k, kBcaThreads, smem, T);
    if (!grid) return RDFFT_E_SHAPE;
    k<<<grid, kBcaThreads, smem, st>>>(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
                                       static_cast<__nv_bfloat16*>(y), T, q_in, q_out, (int)p, logp, acc, wspec);
  }
  return launched();
}

int bca_fwd(const void* x, const void* w, void* y, int64_t T, int64_t d_in, int64_t d_out, int64_t p, int dtype,
            void* stream) {
  return bca_fwd_impl(x, w, y, T, d_in, d_out, p, dtype, stream, 0);
}

int bca_fwd_accum(const void* x, const void* w, void* y, int64_t T, int64_t d_in, int64_t d_out, int64_t p,
                  int dtype, void* stream) {
  return bca_fwd_impl(x, w, y, T, d_in, d_out, p, dtype, stream, 1);
}

int bca_fwd_spectral(const void* x, const float* W, void* y, int64_t T, int64_t d_in, int64_t d_out, int64_t p,
                     int dtype, int accumulate, void* stream) {
  if (!W) return T == 0 ? RDFFT_OK : RDFFT_E_NULL;
  return bca_fwd_impl(x, nullptr, y, T, d_in, d_out, p, dtype, stream, accumulate ? 1 : 0, W);
}

// wspec: resident weight spectra instead of w; spectral_dw: leave dw as accumulated packed spectra
// (no finalize inverse) — the spectral-domain gradient of the resident spectra.
static int bca_bwd_impl(const void* x, const void* w, const void* g, void* dx, float* dw, int64_t T, int64_t d_in,
                 int64_t d_out, int64_t p, int dtype, void* stream, bool accumulate, const float* wspec = nullptr,
                 bool spectral_dw = false) {
  if (wspec) w = wspec;
  int rc = bca_check(x, w, T, d_in, d_out, p, dtype);
  if (rc != RDFFT_OK) return rc;
  if (!dw) return RDFFT_E_NULL;
  if (!aligned16(dw)) return RDFFT_E_ALIGN;
  const size_t s = dsize(dtype);
  const int q_in = (int)(d_in / p), q_out = (int)(d_out / p);
  const size_t nw = (size_t)q_out * q_in * p;
  const size_t xb = T * d_in * s, gb = T * d_out * s;
  const size_t ws = wspec ? 4 : s;
  if (T > 0) {
    if (!g || !dx) return RDFFT_E_NULL;
    if (!aligned16(g) || !aligned16(dx)) return RDFFT_E_ALIGN;
    if (overlap(dx, xb, x, xb) || overlap(dx, xb, w, nw * ws)) return RDFFT_E_ALIAS;
    if (overlap(dx, xb, g, gb) && !(dx == g && d_in == d_out)) return RDFFT_E_ALIAS;
  }
  if (overlap(dw, nw * 4, x, xb) || overlap(dw, nw * 4, w, nw * ws) || overlap(dw, nw * 4, g, gb) ||
      overlap(dw, nw * 4, dx, xb))
    return RDFFT_E_ALIAS;
  const size_t smem = bca_bwd_smem_floats(q_in, q_out, (int)p) * sizeof(float);
  const bool tiled = smem > 227 * 1024;
  BcaTiledPlan plan{};
  if (tiled && !bca_tiled_plan(true, dx == g, T, q_in, q_out, (int)p, num_sms(), &plan)) return RDFFT_E_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (accumulate && spectral_dw) {
    // dW already holds spectra: the kernels add this call's on top
  } else if (accumulate) {  // old dw -> its spectra; the kernels add theirs; the finalize inverse returns old + new
    if ((rc = launch_transform<float>(dw, (int64_t)q_out * q_in, (int)p, /*inverse=*/false, st)) != RDFFT_OK)
      return rc;
  } else if (cudaMemsetAsync(dw, 0, nw * sizeof(float), st) != cudaSuccess) {
    return RDFFT_E_CUDA;
  }
  const int logp = ilog2(p);
  if (tiled && T > 0) {
    const dim3 grid((unsigned)std::min<int64_t>(plan.tiles, (int64_t)num_sms() * 4), (unsigned)plan.groups);
    if (dtype == RDFFT_F32) {
      auto k = bca_bwd_tiled_kernel<float>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
      k<<<grid, kBcaTiledThreads, plan.smem, st>>>(static_cast<const float*>(x), static_cast<const float*>(w),
                                                    static_cast<const float*>(g), static_cast<float*>(dx), dw, T,
                                                    q_in, q_out, (int)p, logp, plan.vt, plan.grp, wspec);
    } else {
      auto k = bca_bwd_tiled_kernel<__nv_bfloat16>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
      k<<<grid, kBcaTiledThreads, plan.smem, st>>>(
          static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
          static_cast<const __nv_bfloat16*>(g), static_cast<__nv_bfloat16*>(dx), dw, T, q_in, q_out, (int)p, logp,
          plan.vt, plan.grp, wspec);
    }
    if ((rc = launched()) != RDFFT_OK) return rc;
    if (spectral_dw) return RDFFT_OK;
    return launch_transform<float>(dw, (int64_t)q_out * q_in, (int)p, /*inverse=*/true, st);
  }
  const bool fast =
      !tiled && T > 0 && (dtype == RDFFT_F32
                    ? bca_bwd_fast<float>(static_cast<const float*>(x), static_cast<const float*>(w),
                                          static_cast<const float*>(g), static_cast<float*>(dx), dw, T, q_in, q_out,
                                          (int)p, num_sms(), st, wspec)
                    : bca_bwd_fast<__nv_bfloat16>(
                          static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
                          static_cast<const __nv_bfloat16*>(g), static_cast<__nv_bfloat16*>(dx), dw, T, q_in, q_out,
                          (int)p, num_sms(), st, wspec));
  if (fast) {
    if ((rc = launched()) != RDFFT_OK) return rc;
  } else if (T > 0 && !tiled) {
    if (dtype == RDFFT_F32) {
      auto k = bca_bwd_v1_kernel<float>;
      const int grid = grid_for(k, kBcaThreads, smem, T);
      if (!grid) return RDFFT_E_SHAPE;
      k<<<grid, kBcaThreads, smem, st>>>(static_cast<const float*>(x), static_cast<const float*>(w),
                                         static_cast<const float*>(g), static_cast<float*>(dx), dw, T, q_in, q_out,
                                         (int)p, logp, wspec);
    } else {
      auto k = bca_bwd_v1_kernel<__nv_bfloat16>;
      const int grid = grid_for(k, kBcaThreads, smem, T);
      if (!grid) return RDFFT_E_SHAPE;
      k<<<grid, kBcaThreads, smem, st>>>(static_cast<const __nv_bfloat16*>(x),
                                         static_cast<const __nv_bfloat16*>(w), static_cast<const __nv_bfloat16*>(g),
                                         static_cast<__nv_bfloat16*>(dx), dw, T, q_in, q_out, (int)p, logp, wspec);
    }
    if ((rc = launched()) != RDFFT_OK) return rc;
  }
  if (spectral_dw) return RDFFT_OK;
  // dw finalise: in-place inverse rdFFT of the q_out*q_in accumulated fp32 spectra.
  return launch_transform<float>(dw, (int64_t)q_out * q_in, (int)p, /*inverse=*/true, st);
}

int bca_bwd(const void* x, const void* w, const void* g, void* dx, float* dw, int64_t T, int64_t d_in, int64_t d_out,
            int64_t p, int dtype, void* stream) {
  return bca_bwd_impl(x, w, g, dx, dw, T, d_in, d_out, p, dtype, stream, false);
}

int bca_bwd_accum(const void* x, const void* w, const void* g, void* dx, float* dw, int64_t T, int64_t d_in,
                  int64_t d_out, int64_t p, int dtype, void* stream) {
  return bca_bwd_impl(x, w, g, dx, dw, T, d_in, d_out, p, dtype, stream, true);
}

int bca_bwd_spectral(const void* x, const float* W, const void* g, void* dx, float* dW, int64_t T, int64_t d_in,
                     int64_t d_out, int64_t p, int dtype, int accumulate, void* stream) {
  if (!W) return RDFFT_E_NULL;
  return bca_bwd_impl(x, nullptr, g, dx, dW, T, d_in, d_out, p, dtype, stream, accumulate != 0, W, true);
}

int rdfft_filter_host(void* xh, int64_t batch, int64_t n, int dtype, const void* filt, int conj, void* work,
                      int64_t work_rows, void* stream0, void* stream1) {
  if (dtype != RDFFT_F32 && dtype != RDFFT_BF16) return RDFFT_E_DTYPE;
  if (!pow2_transform(n)) return RDFFT_E_SIZE;
  if (batch < 0 || work_rows < 2) return RDFFT_E_SHAPE;
  if (batch == 0) return RDFFT_OK;
  if (!xh || !work) return RDFFT_E_NULL;
  if (!aligned16(work) || (filt && !aligned16(filt))) return RDFFT_E_ALIGN;
  const size_t s = dsize(dtype);
  const int64_t half = work_rows / 2;
  const size_t row_bytes = (size_t)n * s;
  if (filt && overlap(filt, row_bytes, work, (size_t)work_rows * row_bytes)) return RDFFT_E_ALIAS;
  cudaStream_t st[2] = {static_cast<cudaStream_t>(stream0), static_cast<cudaStream_t>(stream1)};
  char* host = static_cast<char*>(xh);
  int rc = RDFFT_OK;
  for (int64_t lo = 0, c = 0; lo < batch; lo += half, ++c) {
    const int64_t rows = batch - lo < half ? batch - lo : half;
    cudaStream_t sc = st[c & 1];
    char* dev = static_cast<char*>(work) + (size_t)(c & 1) * half * row_bytes;
    const size_t bytes = (size_t)rows * row_bytes;
    if (cudaMemcpyAsync(dev, host + (size_t)lo * row_bytes, bytes, cudaMemcpyHostToDevice, sc) != cudaSuccess)
      return RDFFT_E_CUDA;
    if ((rc = transform(dev, rows, n, dtype, sc, false)) != RDFFT_OK) return rc;
    if (filt && (rc = packed(dev, filt, rows, n, 1, dtype, sc, conj != 0)) != RDFFT_OK) return rc;
    if ((rc = transform(dev, rows, n, dtype, sc, true)) != RDFFT_OK) return rc;
    if (cudaMemcpyAsync(host + (size_t)lo * row_bytes, dev, bytes, cudaMemcpyDeviceToHost, sc) != cudaSuccess)
      return RDFFT_E_CUDA;
  }
  return RDFFT_OK;
}

const char* rdfft_status_str(int status) {
  switch (status) {
    case RDFFT_OK: return "ok";
    case RDFFT_E_SIZE: return "n is not a power of two in [2, 65536] (BCA block p: [2, 4096])";
    case RDFFT_E_NULL: return "null pointer";
    case RDFFT_E_ALIGN: return "pointer not 16-byte aligned";
    case RDFFT_E_DTYPE: return "unsupported dtype";
    case RDFFT_E_SHAPE: return "invalid shape";
    case RDFFT_E_ALIAS: return "forbidden buffer overlap";
    case RDFFT_E_CUDA: return "CUDA launch error";
    default: return "unknown status";
  }
}

uint64_t rdfft_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int rdfft_abi_version(void) { return 104; }

}  // extern "C"
