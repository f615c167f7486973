// kernels_v1.cuh — packed (conj-)multiply kernels: the TMA-ring kernel for n >= 16
// and a plain staged kernel for n < 16.
#pragma once

#include "stages.cuh"

namespace rdfft {

// a <- a (.) b or a (.) conj(b) per bin; b broadcast when b_batch == 1.
// One CTA row-loop: rows are staged through shared memory with 16-byte global accesses,
// bins are combined from shared memory (slot k with slot n-k), then written back.
constexpr int kPmThreads = 256;
constexpr int kPmTileBytes = 16384;

template <typename T, bool kConj>
__global__ void __launch_bounds__(kPmThreads) packed_mul_kernel(T* __restrict__ a, const T* __restrict__ b,
                                                                int64_t batch, int n, int logn, int64_t b_batch) {
  constexpr int VEC = io<T>::kVec;
  __shared__ __align__(16) unsigned char sa_raw[kPmTileBytes];
  __shared__ __align__(16) unsigned char sb_raw[kPmTileBytes];
  T* sa = reinterpret_cast<T*>(sa_raw);
  T* sbv = reinterpret_cast<T*>(sb_raw);
  const int rows = kPmTileBytes / (int)sizeof(T) >> logn;  // rows per tile (>= 1 for n <= 4096 f32)
  const int64_t ntiles = (batch + rows - 1) / rows;
  const bool bcast = (b_batch == 1);
  const int half = n >> 1;
  if (bcast) {  // the broadcast spectrum is staged once per CTA
    for (int i = threadIdx.x; i < n; i += blockDim.x) sbv[i] = b[i];
  }
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * rows;
    const int nr = (int)(batch - r0 < rows ? batch - r0 : rows);
    const int cnt = nr * n;
    T* ag = a + r0 * n;
    const T* bg = b + r0 * n;
    __syncthreads();
    const int nvec = (cnt % VEC == 0) ? cnt / VEC : 0;
    for (int q = threadIdx.x; q < nvec; q += blockDim.x) {
      reinterpret_cast<uint4*>(sa)[q] = __ldcs(reinterpret_cast<const uint4*>(ag) + q);
      if (!bcast) reinterpret_cast<uint4*>(sbv)[q] = __ldcs(reinterpret_cast<const uint4*>(bg) + q);
    }
    for (int i = nvec * VEC + threadIdx.x; i < cnt; i += blockDim.x) {
      sa[i] = ag[i];
      if (!bcast) sbv[i] = bg[i];
    }
    __syncthreads();
    for (int it = threadIdx.x; it < nr * half; it += blockDim.x) {
      const int r = it >> (logn - 1), k = it & (half - 1);
      T* ar = sa + (r << logn);
      const T* br = sbv + (bcast ? 0 : (r << logn));
      if (k == 0) {  // DC and Nyquist are real
        io<T>::st(ar, io<T>::ld(ar) * io<T>::ld(br));
        io<T>::st(ar + half, io<T>::ld(ar + half) * io<T>::ld(br + half));
      } else {
        const float2 A = make_float2(io<T>::ld(ar + k), io<T>::ld(ar + n - k));
        const float2 B = make_float2(io<T>::ld(br + k), io<T>::ld(br + n - k));
        const float2 C = kConj ? cmulc(A, B) : cmul(A, B);
        io<T>::st(ar + k, C.x);
        io<T>::st(ar + n - k, C.y);
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nvec; q += blockDim.x)
      __stcs(reinterpret_cast<uint4*>(ag) + q, reinterpret_cast<const uint4*>(sa)[q]);
    for (int i = nvec * VEC + threadIdx.x; i < cnt; i += blockDim.x) ag[i] = sa[i];
  }
}

// ---------------------------------------------------------------------------------------------
// packed_mul2 (n >= 16): persistent, TMA-pipelined.  Raw tiles of a (and b unless broadcast) are
// bulk-copied into a ring of shared-memory stages, combined in place bin by bin (slot k with slot
// n-k), and bulk-copied back; the CTA only issues shared-memory instructions.
constexpr int kPm2Threads = 256;
constexpr int kPm2TileBytes = 16384;
constexpr int kPm2Stages = 3;

template <typename T, bool kConj>
__global__ void __launch_bounds__(kPm2Threads) packed_mul2_kernel(T* __restrict__ a, const T* __restrict__ b,
                                                                  int64_t batch, int n, int logn, int64_t b_batch) {
  extern __shared__ float4 pm2_smem[];
  unsigned char* base = reinterpret_cast<unsigned char*>(pm2_smem);
  const bool bcast = (b_batch == 1);
  // [a stages][b stages or one broadcast row][bars: a stages + b stages + 1]
  unsigned char* sa = base;
  unsigned char* sb = base + kPm2Stages * kPm2TileBytes;
  const size_t b_bytes = bcast ? (size_t)n * sizeof(T) : (size_t)kPm2Stages * kPm2TileBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + ((b_bytes + 15) & ~(size_t)15));
  const int rows = (kPm2TileBytes / (int)sizeof(T)) >> logn;
  const int64_t ntiles = (batch + rows - 1) / rows;
  const int half = n >> 1;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < 2 * kPm2Stages + 1; ++s) mbar_init(bar + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto tile_bytes = [&](int64_t t) {
    const int64_t nr = batch - t * rows < rows ? batch - t * rows : rows;
    return (uint32_t)(nr * n * (int)sizeof(T));
  };
  auto issue = [&](int64_t t, int s) {
    fence_proxy_async_smem();
    const uint32_t by = tile_bytes(t);
    mbar_arrive_expect_tx(bar + s, bcast ? by : 2 * by);
    bulk_g2s(sa + s * kPm2TileBytes, a + t * rows * (int64_t)n, by, bar + s);
    if (!bcast) bulk_g2s(sb + s * kPm2TileBytes, b + t * rows * (int64_t)n, by, bar + s);
  };
  if (tid == 0) {
    if (bcast) {
      mbar_arrive_expect_tx(bar + 2 * kPm2Stages, (uint32_t)(n * sizeof(T)));
      bulk_g2s(sb, b, (uint32_t)(n * sizeof(T)), bar + 2 * kPm2Stages);
    }
    for (int s = 0; s < kPm2Stages - 1; ++s) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  }
  if (bcast) mbar_wait(bar + 2 * kPm2Stages, 0);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % kPm2Stages;
    // keep kPm2Stages - 1 loads in flight: refill the stage whose store was issued last iteration
    if (tid == 0) {
      const int64_t t2 = tile + (int64_t)(kPm2Stages - 1) * gridDim.x;
      if (t2 < ntiles) {
        bulk_wait_read<0>();  // the store that last read stage (it + S - 1) % S has drained its source
        issue(t2, (it + kPm2Stages - 1) % kPm2Stages);
      }
    }
    mbar_wait(bar + s, (it / kPm2Stages) & 1);
    const int nr = (int)(batch - tile * rows < rows ? batch - tile * rows : rows);
    T* ta = reinterpret_cast<T*>(sa + s * kPm2TileBytes);
    const T* tb = reinterpret_cast<const T*>(bcast ? sb : sb + s * kPm2TileBytes);
    for (int e = tid; e < (nr << (logn - 1)); e += kPm2Threads) {
      const int r = e >> (logn - 1), k = e & (half - 1);
      T* ar = ta + (r << logn);
      const T* br = tb + (bcast ? 0 : (r << logn));
      if (k == 0) {  // DC and Nyquist are real
        io<T>::st(ar, io<T>::ld(ar) * io<T>::ld(br));
        io<T>::st(ar + half, io<T>::ld(ar + half) * io<T>::ld(br + half));
      } else {
        const float2 A = make_float2(io<T>::ld(ar + k), io<T>::ld(ar + n - k));
        const float2 B = make_float2(io<T>::ld(br + k), io<T>::ld(br + n - k));
        const float2 C = kConj ? cmulc(A, B) : cmul(A, B);
        io<T>::st(ar + k, C.x);
        io<T>::st(ar + n - k, C.y);
      }
    }
    fence_proxy_async_smem();  // generic-proxy writes -> visible to the bulk store
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(a + tile * rows * (int64_t)n, ta, tile_bytes(tile));
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait<0>();
}

}  // namespace rdfft
