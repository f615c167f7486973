// bca_tiled.cuh — BCA forward / backward for layers whose weight spectra do not fit on chip.
//
// Same mathematics as bca_v1.cuh (Eq. 4 / Eq. 5; reading C11), for any
// q_out x q_in: e.g. the D = 4096, p = 128 layer of Tab. 1 has
// q^2 p = 131072 weight taps (512 KB of fp32 spectra).  Instead of keeping every
// W_ij = rdFFT(w_ij) resident, a CTA owns a tile of VT tokens and one group of
// output blocks i (forward) or input blocks j (backward) and transforms the weight
// rows it needs on the fly, once per tile; x / g / y / dx still cross HBM once per
// group and the library allocates nothing.  dw spectra are accumulated straight
// into the caller's fp32 dw with atomics (one per slot per tile) and finalised by
// the same in-place inverse transform as the other paths.
#pragma once

#include "stages.cuh"

namespace rdfft {

constexpr int kBcaTiledThreads = 512;
constexpr size_t kBcaTiledSmemBudget = 200 * 1024;

// shared-memory floats for a tile of vt tokens and a block group of size grp
__host__ __device__ constexpr size_t bca_tiled_fwd_floats(int vt, int q_in, int p) {
  return (size_t)p + (size_t)vt * q_in * p + (size_t)q_in * p + (size_t)vt * p;
}
__host__ __device__ constexpr size_t bca_tiled_bwd_floats(int vt, int grp, int q_out, int p) {
  (void)q_out;
  return (size_t)p + 2 * (size_t)vt * grp * p + (size_t)grp * p + (size_t)vt * p;
}

// Forward: CTA (tile, group): X_vj for all j of the tile's tokens, then for each
// output block i of the group: W_i. = rdFFT(w_i.), Y_v = sum_j W_ij (.) X_vj, y_vi = IrdFFT(Y_v).
template <typename T>
__global__ void __launch_bounds__(kBcaTiledThreads) bca_fwd_tiled_kernel(const T* __restrict__ x,
                                                                         const T* __restrict__ w,
                                                                         T* __restrict__ y, int64_t T_, int q_in,
                                                                         int q_out, int p, int logp, int vt,
                                                                         int grp, int yacc,
                                                                         const float* __restrict__ wspec) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  float2* tw = reinterpret_cast<float2*>(smem);
  float* X = smem + p;                         // [vt][q_in][p]
  float* Wr = X + (size_t)vt * q_in * p;       // [q_in][p]
  float* Y = Wr + (size_t)q_in * p;            // [vt][p]
  make_twiddles(tw, p);
  const int hb = p >> 1;
  const int64_t d_in = (int64_t)q_in * p, d_out = (int64_t)q_out * p;
  const int i0 = blockIdx.y * grp, i1 = min(q_out, i0 + grp);
  const int ntiles = (int)((T_ + vt - 1) / vt);  // 32-bit tile indices (T < 2^31 tokens)
  __syncthreads();
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t t0 = (int64_t)tile * vt;
    const int nv = (int)(T_ - t0 < vt ? T_ - t0 : vt);
    load_rows<T>(x + t0 * d_in, X, nv * q_in * p, p, logp, /*rev=*/true);
    __syncthreads();
    fwd_stages_smem(X, nv * q_in, p, logp, tw);
    for (int i = i0; i < i1; ++i) {
      if (wspec) {  // resident spectra: copy row block i
        load_rows<float>(wspec + (int64_t)i * d_in, Wr, q_in * p, p, logp, /*rev=*/false);
        __syncthreads();
      } else {
        load_rows<T>(w + (int64_t)i * d_in, Wr, q_in * p, p, logp, /*rev=*/true);
        __syncthreads();
        fwd_stages_smem(Wr, q_in, p, logp, tw);
      }
      for (int it = threadIdx.x; it < nv * hb; it += blockDim.x) {
        const int v = it >> (logp - 1);  // hb = p / 2 is a power of two: no integer division
        const PackedBin bin{p, it & (hb - 1)};
        float2 acc = make_float2(0.f, 0.f);
        for (int j = 0; j < q_in; ++j) {
          const float2 prod = bin.mul(bin.get(Wr + (size_t)j * p), bin.get(X + ((size_t)v * q_in + j) * p));
          acc.x += prod.x;
          acc.y += prod.y;
        }
        bin.put(Y + (size_t)v * p, acc);
      }
      __syncthreads();
      inv_stages_smem(Y, nv, p, logp, tw);
      for (int v = 0; v < nv; ++v)
        store_rows<T>(y + (t0 + v) * d_out + (int64_t)i * p, Y + (size_t)v * p, p, p, logp, /*rev=*/true,
                      yacc != 0);
      __syncthreads();
    }
  }
}

// Backward: CTA (tile, group of input blocks j in [j0, j1)): X_vj for its j, then for each
// output block i: G_vi = rdFFT(g_vi), W_ij = rdFFT(w_ij) for its j,
//   D_vj += conj(W_ij) (.) G_vi,   dw_ij += sum_v conj(X_vj) (.) G_vi  (fp32 atomics),
// and finally dx_vj = IrdFFT(D_vj).  All g reads of a tile precede its dx writes, so dx may be g.
template <typename T>
__global__ void __launch_bounds__(kBcaTiledThreads) bca_bwd_tiled_kernel(const T* __restrict__ x,
                                                                         const T* __restrict__ w, const T* g, T* dx,
                                                                         float* __restrict__ dw, int64_t T_,
                                                                         int q_in, int q_out, int p, int logp,
                                                                         int vt, int grp,
                                                                         const float* __restrict__ wspec) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  float2* tw = reinterpret_cast<float2*>(smem);
  const int j0 = blockIdx.y * grp, ng = min(q_in, j0 + grp) - j0;
  float* X = smem + p;                        // [vt][ng][p]
  float* D = X + (size_t)vt * grp * p;        // [vt][ng][p]
  float* WG = D + (size_t)vt * grp * p;       // W_i,j0.. [ng][p] then G_v [vt][p] (one transform batch)
  float* G = WG + (size_t)ng * p;
  make_twiddles(tw, p);
  const int hb = p >> 1;
  const int64_t d_in = (int64_t)q_in * p, d_out = (int64_t)q_out * p;
  const int64_t ntiles = (T_ + vt - 1) / vt;
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t t0 = tile * vt;
    const int nv = (int)(T_ - t0 < vt ? T_ - t0 : vt);
    for (int v = 0; v < nv; ++v)
      load_rows<T>(x + (t0 + v) * d_in + (int64_t)j0 * p, X + (size_t)v * ng * p, ng * p, p, logp, true);
    for (int e = threadIdx.x; e < nv * ng * p; e += blockDim.x) D[e] = 0.f;
    __syncthreads();
    fwd_stages_smem(X, nv * ng, p, logp, tw);
    for (int i = 0; i < q_out; ++i) {
      if (wspec)
        load_rows<float>(wspec + ((int64_t)i * q_in + j0) * p, WG, ng * p, p, logp, false);
      else
        load_rows<T>(w + ((int64_t)i * q_in + j0) * p, WG, ng * p, p, logp, true);
      for (int v = 0; v < nv; ++v) load_rows<T>(g + (t0 + v) * d_out + (int64_t)i * p, G + (size_t)v * p, p, p, logp, true);
      __syncthreads();
      if (wspec)
        fwd_stages_smem(G, nv, p, logp, tw);
      else
        fwd_stages_smem(WG, ng + nv, p, logp, tw);
      for (int it = threadIdx.x; it < ng * hb; it += blockDim.x) {
        const int j = it / hb;
        const PackedBin bin{p, it - j * hb};
        const float2 wij = bin.get(WG + (size_t)j * p);
        float2 acc = make_float2(0.f, 0.f);
        for (int v = 0; v < nv; ++v) {
          const float2 gv = bin.get(G + (size_t)v * p);
          float* d = D + ((size_t)v * ng + j) * p;
          const float2 dd = bin.mulc(gv, wij);
          const float2 cur = bin.get(d);
          bin.put(d, make_float2(cur.x + dd.x, cur.y + dd.y));
          const float2 xg = bin.mulc(gv, bin.get(X + ((size_t)v * ng + j) * p));
          acc.x += xg.x;
          acc.y += xg.y;
        }
        float* a = dw + ((int64_t)i * q_in + j0 + j) * p;
        if (bin.k == 0) {
          atomicAdd(a, acc.x);
          atomicAdd(a + hb, acc.y);
        } else {
          atomicAdd(a + bin.k, acc.x);
          atomicAdd(a + p - bin.k, acc.y);
        }
      }
      __syncthreads();
    }
    inv_stages_smem(D, nv * ng, p, logp, tw);
    for (int v = 0; v < nv; ++v)
      store_rows<T>(dx + (t0 + v) * d_in + (int64_t)j0 * p, D + (size_t)v * ng * p, ng * p, p, logp, true);
    __syncthreads();
  }
}

// Host planning: largest token tile (<= 16) that fits the budget with the whole block range
// in one group; if even vt = 1 does not fit, split the block range.  Then split the block
// range further while the grid has fewer CTAs than SMs.  When dx aliases g (in_place) the
// backward keeps one group: another group's CTA would still read g blocks this one has
// overwritten with dx.
struct BcaTiledPlan {
  int vt, grp, groups;
  int64_t tiles;
  size_t smem;
};

inline bool bca_tiled_plan(bool bwd, bool in_place, int64_t T_, int q_in, int q_out, int p, int sms,
                           BcaTiledPlan* out) {
  const int q = bwd ? q_in : q_out;  // the split dimension
  auto bytes = [&](int vt, int grp) {
    return 4 * (bwd ? bca_tiled_bwd_floats(vt, grp, q_out, p) : bca_tiled_fwd_floats(vt, q_in, p));
  };
  int grp = q, vt = 16;
  while (vt > 1 && bytes(vt, grp) > kBcaTiledSmemBudget) vt >>= 1;
  while (bwd && grp > 1 && bytes(vt, grp) > kBcaTiledSmemBudget) grp = (grp + 1) / 2;
  if (bytes(vt, grp) > 227 * 1024 || (in_place && grp < q)) return false;
  if (T_ < vt) vt = (int)(T_ > 0 ? T_ : 1);
  const int64_t tiles = (T_ + vt - 1) / vt;
  while (!in_place && grp > 1 && tiles * ((q + grp - 1) / grp) < sms) grp = (grp + 1) / 2;
  out->vt = vt;
  out->grp = grp;
  out->groups = (q + grp - 1) / grp;
  out->tiles = tiles;
  out->smem = bytes(vt, grp);
  return true;
}

}  // namespace rdfft
