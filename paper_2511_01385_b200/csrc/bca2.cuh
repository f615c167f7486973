// bca2.cuh — fused block-circulant adapter (BCA) forward / backward on the
// register-blocked 2-pass transform (plan2.cuh); square layers (q_in == q_out
// = q <= 4), p in {256, 512, 1024}.
//
// Forward (Eq. 4; blocks P:L184), per tile of TT tokens
// (TT q consecutive p-blocks = one contiguous tile of the activation):
//   X = rdFFT(x) in shared memory -> Y_i = sum_j W_ij (.) X_j in place ->
//   y = IrdFFT(Y) straight to HBM.
// W_ij = rdFFT(w_ij) is computed once per CTA into a resident shared-memory
// region with the same half-pair layout (reading C12); x is never written (C13).
//
// Backward (Eq. 5; pairing C11), per tile:
//   X = rdFFT(x), G = rdFFT(g) (two thread groups, one per operand)
//   Acc_ij += conj(X_j) (.) G_i     per-thread fp32 registers for the CTA's whole token range
//   D_j = sum_i conj(W_ij) (.) G_i  in place of X_j,  dx = IrdFFT(D)  (dx may alias g)
// then Acc is added to dw with fp32 atomics; dw is zeroed before and
// inverse-transformed after (dw finalize launch), in fp32.
//
// Product layout: item u < N/4 owns half-pair positions u and N/2 - u, i.e. the
// complex bins u and N/2 - u:  bin u = (H[u].x, H[N/2-u].y), bin N/2-u = (H[N/2-u].x, H[u].y).
// Item 0 owns H[0] = (DC, Nyquist) (two real bins) and H[N/4] = bin N/4.
#pragma once

#include "plan2.cuh"

namespace rdfft {

constexpr int kBcaQMax = 4;

// Resident weight-spectra rows: sized for q = kBcaQMax up to p = 1024 (unchanged layouts), for the
// kernel's own q at p >= 2048 (a 4096-point spectrum row is ~17 KB).
template <typename P, int Q>
constexpr int bca_wrows() { return P::N >= 2048 ? Q * Q : kBcaQMax * kBcaQMax; }

template <typename P, int Q = kBcaQMax>
struct BcaFwdSmem {  // [stage x STAGES][H][W][TWf][TWi][bars]; STAGES = 0: pass 1 reads x from HBM
  static constexpr int STAGES = P::NSTG;
  static constexpr int WF = bca_wrows<P, Q>() * P::ROWA + 16;
  static constexpr size_t H_OFF = (size_t)STAGES * P::STAGE;
  static constexpr size_t W_OFF = H_OFF + (size_t)P::HF * 8;
  static constexpr size_t TWF_OFF = W_OFF + (size_t)WF * 8;
  static constexpr size_t TWI_OFF = TWF_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BAR_OFF = TWI_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BYTES = BAR_OFF + 16;
  static_assert(STAGES <= 2, "staging depth");
};

// complex helpers on float2 (re, im)
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 c) {  // c + a b
  return make_float2(fmaf(a.x, b.x, fmaf(-a.y, b.y, c.x)), fmaf(a.x, b.y, fmaf(a.y, b.x, c.y)));
}
__device__ __forceinline__ float2 cfmac(float2 a, float2 b, float2 c) {  // c + conj(a) b
  return make_float2(fmaf(a.x, b.x, fmaf(a.y, b.y, c.x)), fmaf(a.x, b.y, fmaf(-a.y, b.x, c.y)));
}

// Branch-free per-bin multiply-accumulate shared by generic and special items.  The right
// operand b is prepared once (per token) into four values so that every (i, j) pair costs
// exactly 4 FFMA whether the bin pair is complex (c += a b or c += conj(a) b) or the special
// (DC, Nyquist) pair of real bins (c.x += a.x b.x, c.y += a.y b.y):
//   c.x += a.x p + a.y r,   c.y += a.x t + a.y u.
struct PrepB {
  float p, r, t, u;
};
template <bool kConjA>
__device__ __forceinline__ PrepB prep_b(float2 b, bool special) {
  if (special) return {b.x, 0.f, 0.f, b.y};
  return kConjA ? PrepB{b.x, b.y, b.y, -b.x} : PrepB{b.x, -b.y, b.y, b.x};
}
__device__ __forceinline__ float2 pmac(float2 a, const PrepB& b, float2 c) {
  return make_float2(fmaf(a.y, b.r, fmaf(a.x, b.p, c.x)), fmaf(a.y, b.u, fmaf(a.x, b.t, c.y)));
}

// Gather the two bins of item u from the half pairs at positions (pa, pb) of one row.
struct BinPair {
  float2 b1, b2;
};
__device__ __forceinline__ BinPair bins_get(const float2* rowbase, int oa, int ob, bool special) {
  const float2 a = rowbase[oa], b = rowbase[ob];
  if (special) return {a, b};                                    // (DC, Nyq) and bin N/4
  return {make_float2(a.x, b.y), make_float2(b.x, a.y)};
}
__device__ __forceinline__ void bins_put(float2* rowbase, int oa, int ob, bool special, BinPair v) {
  if (special) {
    rowbase[oa] = v.b1;
    rowbase[ob] = v.b2;
  } else {
    rowbase[oa] = make_float2(v.b1.x, v.b2.y);
    rowbase[ob] = make_float2(v.b2.x, v.b1.y);
  }
}

template <typename P>
__device__ __forceinline__ void bca_item_offsets(int u, int& oa, int& ob) {
  // physical float2 offsets (relative to a row) of half-pair positions of item u
  constexpr int R = P::R, W = P::WSTR, HALF = P::N / 2;
  const int qa = u, qb = (u == 0) ? P::N / 4 : HALF - u;
  oa = (qa / R) * W + qa % R;
  ob = (qb / R) * W + qb % R;
}

// In-place forward product over one tile: Y_i = sum_j W_ij (.) X_j for tokens of this tile.
template <typename P, int Q>
__device__ __forceinline__ void bca_product_fwd(float2* H, const float2* Wr, int ntok, int tid) {
  constexpr int q = Q;
  constexpr int NI = P::N / 4;
  constexpr int TS = P::NT >= NI ? P::NT / NI : 1;  // thread groups sharing an item (token split)
  for (int u = tid % NI; u < NI; u += (P::NT >= NI ? NI : P::NT)) {
    const int ts = P::NT >= NI ? tid / NI : 0;
    int oa, ob;
    bca_item_offsets<P>(u, oa, ob);
    const bool special = (u == 0);
    BinPair w[Q][Q];
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int j = 0; j < Q; ++j)
        if (i < q && j < q) w[i][j] = bins_get(Wr + P::row(i * q + j), oa, ob, special);
    for (int tt = ts; tt < ntok; tt += TS) {
      PrepB x1[Q];
      float2 x2[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j)
        if (j < q) {
          const BinPair xb = bins_get(H + P::row(tt * q + j), oa, ob, special);
          x1[j] = prep_b<false>(xb.b1, special);
          x2[j] = xb.b2;
        }
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        if (i < q) {
          BinPair y = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int j = 0; j < Q; ++j) {
            if (j < q) {
              y.b1 = pmac(w[i][j].b1, x1[j], y.b1);
              y.b2 = cfma(w[i][j].b2, x2[j], y.b2);
            }
          }
          bins_put(H + P::row(tt * q + i), oa, ob, special, y);
        }
      }
    }
  }
}

template <typename P, int Q>
__global__ void __launch_bounds__(P::NT, 1) bca_fwd2_kernel(const typename P::elem* __restrict__ x,
                                                         const typename P::elem* __restrict__ w,
                                                         typename P::elem* __restrict__ y, int64_t T_,
                                                         int acc, const float* __restrict__ wspec) {
  constexpr int q = Q;
  using T = typename P::elem;
  using L = BcaFwdSmem<P, Q>;
  constexpr int N = P::N;
  static_assert(Q * Q <= P::VT, "the weight prologue transforms q*q <= VT spectra in one pass");
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float2* H = reinterpret_cast<float2*>(base + L::H_OFF);
  float2* Wr = reinterpret_cast<float2*>(base + L::W_OFF);
  float2* TWf = reinterpret_cast<float2*>(base + L::TWF_OFF);
  float2* TWi = reinterpret_cast<float2*>(base + L::TWI_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  const int tid = threadIdx.x;
  const int TT = P::VT / q;                 // tokens per tile
  const int64_t ntiles = (T_ + TT - 1) / TT;
  const int64_t tok_elems = (int64_t)q * N;  // elements per token row (d = q p)
  p2_tables<P>(TWf, TWi, tid, P::NT);
  p2_zero_pads<P>(H, P::VT, tid, P::NT);
  p2_zero_pads<P>(Wr, q * q, tid, P::NT);
  if (tid == 0) {
    for (int s = 0; s < L::STAGES; ++s) mbar_init(bar + s, 1);
    fence_mbar_init();
  }
  const uint32_t k65536 = kTwo16;
  const P2Roles<P> rh(H, TWf, TWi, tid);
  auto tile_rows = [&](int64_t t) { return (int)((T_ - t * TT < TT ? T_ - t * TT : TT) * q); };
  __syncthreads();
  // the first tiles' TMA loads go out before the weight prologue, so their latency overlaps it (issued
  // after the prologue they added a load latency to every launch; RoBERTa-base forward ~1.5 us)
  if (tid == 0) {
    for (int s = 0; s < L::STAGES; ++s) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < ntiles) stage_issue_rows<P>(x + t * TT * tok_elems, tile_rows(t), base + s * P::STAGE, bar + s);
    }
  }
  // ---- prologue: W_ij = rdFFT(w_ij), q*q <= VT vectors (read straight from HBM), into the resident
  // region (or the caller's resident spectra copied in: wspec)
  if (wspec) {
    p2_load_spectra<P>(Wr, wspec, q * q, tid, P::NT);
  } else {
    const P2Roles<P> rw(Wr, TWf, TWi, tid);
    p2_pass1_fwd<P, true>(rw, w, q * q, k65536);
    __syncthreads();
    p2_last_fwd<P>(rw, q * q);
    p2_dc_fwd<P>(rw, q * q);
  }
  __syncthreads();
  uint32_t phase_use[2] = {0, 0};
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int ntok = (int)(T_ - tile * TT < TT ? T_ - tile * TT : TT);
    const int nv = ntok * q;
    if constexpr (L::STAGES == 0) {
      p2_pass1_fwd<P, true>(rh, x + tile * TT * tok_elems, nv, k65536);
      __syncthreads();
    } else {
      const int sb = L::STAGES == 2 ? (it & 1) : 0;
      const T* st = reinterpret_cast<const T*>(base + sb * P::STAGE);
      mbar_wait(bar + sb, phase_use[sb] & 1);
      ++phase_use[sb];
      p2_pass1_fwd<P>(rh, st, nv, k65536);
      __syncthreads();  // H complete, staging sb consumed
      const int64_t nxt = tile + (int64_t)L::STAGES * gridDim.x;
      if (tid == 0 && nxt < ntiles)
        stage_issue_rows<P>(x + nxt * TT * tok_elems, tile_rows(nxt), base + sb * P::STAGE, bar + sb);
    }
    p2_last_fwd<P>(rh, nv);
    p2_dc_fwd<P>(rh, nv);
    __syncthreads();
    bca_product_fwd<P, Q>(H, Wr, ntok, tid);
    __syncthreads();
    p2_last_inv<P>(rh, nv);
    p2_dc_inv<P>(rh, nv);
    __syncthreads();
    p2_pass1_inv<P>(rh, y + tile * TT * tok_elems, nv, acc != 0);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ backward
template <typename P>
struct BcaBwdSmem {  // [sx x STAGES][sg x STAGES][Hx][Hg][W][TWf][TWi][bars x 2 STAGES]
  static constexpr int STAGES = sizeof(typename P::elem) == 2 ? 2 : 1;
  static constexpr int WF = kBcaQMax * kBcaQMax * P::ROWA + 16;
  static constexpr size_t SG_OFF = (size_t)STAGES * P::STAGE;
  static constexpr size_t HX_OFF = 2 * (size_t)STAGES * P::STAGE;
  static constexpr size_t HG_OFF = HX_OFF + (size_t)P::HF * 8;
  static constexpr size_t W_OFF = HG_OFF + (size_t)P::HF * 8;
  static constexpr size_t TWF_OFF = W_OFF + (size_t)WF * 8;
  static constexpr size_t TWI_OFF = TWF_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BAR_OFF = TWI_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BYTES = BAR_OFF + 32;
};

template <typename P, int Q>
__global__ void __launch_bounds__(2 * P::NT) bca_bwd2_kernel(const typename P::elem* __restrict__ x,
                                                             const typename P::elem* __restrict__ w,
                                                             const typename P::elem* g, typename P::elem* dx,
                                                             float* __restrict__ dw, int64_t T_,
                                                             const float* __restrict__ wspec) {
  constexpr int q = Q;
  using T = typename P::elem;
  using L = BcaBwdSmem<P>;
  constexpr int N = P::N, NT2 = 2 * P::NT, NI = N / 4;
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float2* Hx = reinterpret_cast<float2*>(base + L::HX_OFF);
  float2* Hg = reinterpret_cast<float2*>(base + L::HG_OFF);
  float2* Wr = reinterpret_cast<float2*>(base + L::W_OFF);
  float2* TWf = reinterpret_cast<float2*>(base + L::TWF_OFF);
  float2* TWi = reinterpret_cast<float2*>(base + L::TWI_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);  // [x s0, x s1, g s0, g s1]
  const int tid = threadIdx.x;
  const int grp = tid / P::NT, lt = tid % P::NT;  // group 0: x operand, group 1: g operand
  const int TT = P::VT / q;
  const int64_t ntiles = (T_ + TT - 1) / TT;
  const int64_t tok_elems = (int64_t)q * N;
  unsigned char* stg = base + (grp ? L::SG_OFF : 0);
  uint64_t* gbar = bar + grp * 2;
  const T* src = grp ? g : x;
  float2* Hm = grp ? Hg : Hx;
  p2_tables<P>(TWf, TWi, tid, NT2);
  p2_zero_pads<P>(Hx, P::VT, tid, NT2);
  p2_zero_pads<P>(Hg, P::VT, tid, NT2);
  p2_zero_pads<P>(Wr, q * q, tid, NT2);
  if (tid == 0) {
    for (int s = 0; s < 4; ++s) mbar_init(bar + s, 1);
    fence_mbar_init();
  }
  const uint32_t k65536 = kTwo16;
  const P2Roles<P> rh(Hm, TWf, TWi, lt);
  auto tile_rows = [&](int64_t t) { return (int)((T_ - t * TT < TT ? T_ - t * TT : TT) * q); };
  __syncthreads();
  // ---- prologue: W_ij = rdFFT(w_ij) into the resident region.  q*q <= VT: group 0 does all
  // rows; q*q = 16 > VT = 8: rows [0, 8) by group 0 and [8, 16) by group 1 (8 = skew period,
  // so row(8 + v) == 8 ROWA + row(v)).
  const int nw = q * q;
  const int half = nw <= P::VT ? nw : 8;
  const int w0 = grp ? half : 0, wn = grp ? nw - half : half;
  if (wspec) {
    p2_load_spectra<P>(Wr, wspec, nw, tid, NT2);
  } else {
    if (lt == 0 && wn > 0) stage_issue_rows<P>(w + (int64_t)w0 * N, wn, stg, gbar);
    if (wn > 0) mbar_wait(gbar, 0);
    const P2Roles<P> rw(Wr + w0 * P::ROWA, TWf, TWi, lt);
    p2_pass1_fwd<P>(rw, reinterpret_cast<const T*>(stg), wn, k65536);
    __syncthreads();
    p2_last_fwd<P>(rw, wn);
    p2_dc_fwd<P>(rw, wn);
  }
  __syncthreads();
  uint32_t phase_use[2] = {(wn > 0 && !wspec) ? 1u : 0u, 0};
  if (lt == 0) {
    for (int s = 0; s < L::STAGES; ++s) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < ntiles) stage_issue_rows<P>(src + t * TT * tok_elems, tile_rows(t), stg + s * P::STAGE, gbar + s);
    }
  }
  // dW accumulators: item u = tid (one item per thread when 2 NT == N/4), all q*q pairs, 2 bins
  static_assert(NT2 % NI == 0 || NI % NT2 == 0, "item mapping");
  constexpr int IPT = NI > NT2 ? NI / NT2 : 1;  // items per thread
  constexpr int TS = NT2 >= NI ? NT2 / NI : 1;   // token split
  BinPair acc[IPT][Q][Q];
#pragma unroll
  for (int a = 0; a < IPT; ++a)
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int j = 0; j < Q; ++j) acc[a][i][j] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int ntok = (int)(T_ - tile * TT < TT ? T_ - tile * TT : TT);
    const int nv = ntok * q;
    const int sb = L::STAGES == 2 ? (it & 1) : 0;
    const T* st = reinterpret_cast<const T*>(stg + sb * P::STAGE);
    mbar_wait(gbar + sb, phase_use[sb] & 1);
    ++phase_use[sb];
    p2_pass1_fwd<P>(rh, st, nv, k65536);
    __syncthreads();
    const int64_t nxt = tile + (int64_t)L::STAGES * gridDim.x;
    if (lt == 0 && nxt < ntiles)
      stage_issue_rows<P>(src + nxt * TT * tok_elems, tile_rows(nxt), stg + sb * P::STAGE, gbar + sb);
    p2_last_fwd<P>(rh, nv);
    p2_dc_fwd<P>(rh, nv);
    __syncthreads();
    // ---- products: Acc += conj(X) G ; D = sum_i conj(W_ij) G_i written over X
#pragma unroll
    for (int a = 0; a < IPT; ++a) {
      const int u = (tid % NI) + a * NT2;
      const int ts = NT2 >= NI ? tid / NI : 0;
      int oa, ob;
      bca_item_offsets<P>(u, oa, ob);
      const bool special = (u == 0);
      BinPair wv[Q][Q];
#pragma unroll
      for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = 0; j < Q; ++j)
          if (i < q && j < q) wv[i][j] = bins_get(Wr + P::row(i * q + j), oa, ob, special);
      for (int tt = ts; tt < ntok; tt += TS) {
        BinPair xv[Q], gv[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j)
          if (j < q) {
            xv[j] = bins_get(Hx + P::row(tt * q + j), oa, ob, special);
            gv[j] = bins_get(Hg + P::row(tt * q + j), oa, ob, special);
          }
        PrepB g1[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i)
          if (i < q) g1[i] = prep_b<true>(gv[i].b1, special);
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
          for (int j = 0; j < Q; ++j)
            if (i < q && j < q) {
              acc[a][i][j].b1 = pmac(xv[j].b1, g1[i], acc[a][i][j].b1);
              acc[a][i][j].b2 = cfmac(xv[j].b2, gv[i].b2, acc[a][i][j].b2);
            }
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          if (j < q) {
            BinPair d = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int i = 0; i < Q; ++i)
              if (i < q) {
                d.b1 = pmac(wv[i][j].b1, g1[i], d.b1);
                d.b2 = cfmac(wv[i][j].b2, gv[i].b2, d.b2);
              }
            bins_put(Hx + P::row(tt * q + j), oa, ob, special, d);
          }
        }
      }
    }
    __syncthreads();
    // ---- dx = IrdFFT(D): group 0 (the x group owns Hx)
    if (grp == 0) {
      p2_last_inv<P>(rh, nv);
      p2_dc_inv<P>(rh, nv);
    }
    __syncthreads();
    if (grp == 0) p2_pass1_inv<P>(rh, dx + tile * TT * tok_elems, nv);
    __syncthreads();
  }
  // ---- flush dW accumulators (packed slots) into dw with fp32 atomics
#pragma unroll
  for (int a = 0; a < IPT; ++a) {
    const int u = (tid % NI) + a * NT2;
    const int ts = NT2 >= NI ? tid / NI : 0;
    (void)ts;
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        if (i < q && j < q) {
          float* d = dw + (int64_t)(i * q + j) * N;
          const BinPair v = acc[a][i][j];
          if (u == 0) {
            atomicAdd(d + 0, v.b1.x);
            atomicAdd(d + N / 2, v.b1.y);
            atomicAdd(d + N / 4, v.b2.x);
            atomicAdd(d + 3 * N / 4, v.b2.y);
          } else {
            atomicAdd(d + u, v.b1.x);
            atomicAdd(d + N - u, v.b1.y);
            atomicAdd(d + N / 2 - u, v.b2.x);
            atomicAdd(d + N / 2 + u, v.b2.y);
          }
        }
      }
  }
}

template <typename P, typename K>
int bca2_grid(K kernel, int threads, size_t smem, int64_t units, int sms) {
  if (smem > 227 * 1024) return 0;  // configuration does not fit: caller falls back
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  if (per_sm <= 0) return 0;
  if (verbose())
    std::fprintf(stderr, "[rdfft] bca kernel p=%d VT=%d: %zu B smem, %d threads, %d CTAs/SM\n", P::N, P::VT, smem,
                 threads, per_sm);
  return (int)(units < (int64_t)per_sm * sms ? units : (int64_t)per_sm * sms);
}

// ------------------------------------------------------------------ backward, single group
// One thread group of NT = VT * LPV threads transforms the x tile and then the g tile (pass 1
// straight from HBM, no staging), so the product and the dx inverse use every thread; a tile is
// VT / q tokens.  Shared memory: Hx, Hg, W, tables.
template <typename P, int Q = kBcaQMax>
struct BcaBwd3Smem {
  static constexpr int WF = bca_wrows<P, Q>() * P::ROWA + 16;
  static constexpr int NI = P::N / 4;
  static constexpr int IPT = NI > P::NT ? NI / P::NT : 1;  // product items per thread
  // p = 2048 / 4096 (64-point register blocks, 4 or 8 items per thread): the dW accumulators
  // (IPT q^2 bin pairs per thread) live in shared memory, one float4 per (item, i, j) per thread
  // (thread-major: conflict-free 16-byte accesses), instead of registers that spilled
  // (bf16 p = 4096: 255 registers + 268 B of local memory)
  static constexpr bool ACC_SMEM = IPT >= 4;
  static constexpr size_t HX_OFF = 0;
  static constexpr size_t HG_OFF = HX_OFF + (size_t)P::HF * 8;
  static constexpr size_t W_OFF = HG_OFF + (size_t)P::HF * 8;
  static constexpr size_t TWF_OFF = W_OFF + (size_t)WF * 8;
  static constexpr size_t TWI_OFF = TWF_OFF + (size_t)P::TWF * 8;
  static constexpr size_t ACC_OFF = TWI_OFF + (size_t)P::TWF * 8;
  static constexpr size_t TMEM_OFF = ACC_OFF + (ACC_SMEM ? (size_t)IPT * Q * Q * P::NT * 16 : 0);
  static constexpr size_t BYTES = TMEM_OFF + 16;  // + the TMEM address (bca_bwd4)
};

template <typename P, int Q>
__global__ void __launch_bounds__(P::NT, 1) bca_bwd3_kernel(const typename P::elem* __restrict__ x,
                                                            const typename P::elem* __restrict__ w,
                                                            const typename P::elem* g, typename P::elem* dx,
                                                            float* __restrict__ dw, int64_t T_,
                                                            const float* __restrict__ wspec) {
  constexpr int q = Q;
  using T = typename P::elem;
  using L = BcaBwd3Smem<P, Q>;
  static_assert(Q * Q <= P::VT, "the weight prologue transforms q*q <= VT spectra in one pass");
  constexpr int N = P::N, NT = P::NT, NI = N / 4;
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float2* Hx = reinterpret_cast<float2*>(base + L::HX_OFF);
  float2* Hg = reinterpret_cast<float2*>(base + L::HG_OFF);
  float2* Wr = reinterpret_cast<float2*>(base + L::W_OFF);
  float2* TWf = reinterpret_cast<float2*>(base + L::TWF_OFF);
  float2* TWi = reinterpret_cast<float2*>(base + L::TWI_OFF);
  const int tid = threadIdx.x;
  const int TT = P::VT / q;
  // 32-bit tile indices (T < 2^31 tokens): smaller loop state for the 64-point register blocks
  const int ntiles = (int)((T_ + TT - 1) / TT);
  const int64_t tok_elems = (int64_t)q * N;
  p2_tables<P>(TWf, TWi, tid, NT);
  p2_zero_pads<P>(Hx, P::VT, tid, NT);
  p2_zero_pads<P>(Hg, P::VT, tid, NT);
  p2_zero_pads<P>(Wr, q * q, tid, NT);
  const uint32_t k65536 = kTwo16;
  // one role set: the g group's H region is the x group's shifted by HF (Hg = Hx + HF), so rg is rx
  // with an offset (a second set of role pointers cost ~20 live registers: spills at p = 2048 / 4096)
  const P2Roles<P> rx(Hx, TWf, TWi, tid);
  static_assert(L::HG_OFF == L::HX_OFF + (size_t)P::HF * 8, "Hg = Hx + HF");
  constexpr int GOFF = P::HF;
  __syncthreads();
  if (wspec) {
    p2_load_spectra<P>(Wr, wspec, q * q, tid, NT);
  } else {  // W_ij = rdFFT(w_ij): q*q <= VT vectors
    const P2Roles<P> rw(Wr, TWf, TWi, tid);
    p2_pass1_fwd<P, true>(rw, w, q * q, k65536);
    __syncthreads();
    p2_last_fwd<P>(rw, q * q);
    p2_dc_fwd<P>(rw, q * q);
  }
  __syncthreads();
  static_assert(NT % NI == 0 || NI % NT == 0, "item mapping");
  constexpr int IPT = NI > NT ? NI / NT : 1;  // items per thread
  constexpr int TS = NT >= NI ? NT / NI : 1;   // token split
  static_assert(IPT == L::IPT, "layout");
  constexpr bool kAccS = L::ACC_SMEM;
  float4* accS = reinterpret_cast<float4*>(base + L::ACC_OFF);  // [a][i][j][tid] (kAccS)
  auto acc_slot = [&](int a, int i, int j) { return accS + ((a * Q + i) * Q + j) * NT + tid; };
  BinPair acc[kAccS ? 1 : IPT][Q][Q];
#pragma unroll
  for (int a = 0; a < (kAccS ? 1 : IPT); ++a)
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int j = 0; j < Q; ++j) acc[a][i][j] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  if constexpr (kAccS) {
#pragma unroll
    for (int a = 0; a < IPT; ++a)
#pragma unroll
      for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = 0; j < Q; ++j)
          if (i < q && j < q) *acc_slot(a, i, j) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int ntok = (int)(T_ - (int64_t)tile * TT < TT ? T_ - (int64_t)tile * TT : TT);
    const int nv = ntok * q;
    const int64_t e0 = (int64_t)tile * TT * tok_elems;
    // (compiler fences between the two operands: interleaving two 64-point register FFTs would
    // double the live registers at p = 2048 / 4096)
    p2_pass1_fwd<P, true>(rx, x + e0, nv, k65536);
    asm volatile("" ::: "memory");
    p2_pass1_fwd<P, true>(rx, g + e0, nv, k65536, GOFF);
    __syncthreads();
    p2_last_fwd<P>(rx, nv);
    asm volatile("" ::: "memory");
    p2_last_fwd<P>(rx, nv, GOFF);
    p2_dc_fwd<P>(rx, nv);
    p2_dc_fwd<P>(rx, nv, GOFF);
    __syncthreads();
#pragma unroll
    for (int a = 0; a < IPT; ++a) {
      const int u = (tid % NI) + a * NT;
      const int ts = NT >= NI ? tid / NI : 0;
      int oa, ob;
      bca_item_offsets<P>(u, oa, ob);
      const bool special = (u == 0);
      BinPair wv[Q][Q];
#pragma unroll
      for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = 0; j < Q; ++j)
          if (i < q && j < q) wv[i][j] = bins_get(Wr + P::row(i * q + j), oa, ob, special);
      BinPair (&ac)[Q][Q] = acc[kAccS ? 0 : a];
      if constexpr (kAccS) {
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
          for (int j = 0; j < Q; ++j)
            if (i < q && j < q) {
              const float4 f = *acc_slot(a, i, j);
              ac[i][j] = {make_float2(f.x, f.y), make_float2(f.z, f.w)};
            }
      }
      for (int tt = ts; tt < ntok; tt += TS) {
        BinPair xv[Q], gv[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j)
          if (j < q) {
            xv[j] = bins_get(Hx + P::row(tt * q + j), oa, ob, special);
            gv[j] = bins_get(Hg + P::row(tt * q + j), oa, ob, special);
          }
        PrepB g1[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i)
          if (i < q) g1[i] = prep_b<true>(gv[i].b1, special);
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
          for (int j = 0; j < Q; ++j)
            if (i < q && j < q) {
              ac[i][j].b1 = pmac(xv[j].b1, g1[i], ac[i][j].b1);
              ac[i][j].b2 = cfmac(xv[j].b2, gv[i].b2, ac[i][j].b2);
            }
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          if (j < q) {
            BinPair d = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int i = 0; i < Q; ++i)
              if (i < q) {
                d.b1 = pmac(wv[i][j].b1, g1[i], d.b1);
                d.b2 = cfmac(wv[i][j].b2, gv[i].b2, d.b2);
              }
            bins_put(Hx + P::row(tt * q + j), oa, ob, special, d);
          }
        }
      }
      if constexpr (kAccS) {
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
          for (int j = 0; j < Q; ++j)
            if (i < q && j < q) *acc_slot(a, i, j) = make_float4(ac[i][j].b1.x, ac[i][j].b1.y, ac[i][j].b2.x, ac[i][j].b2.y);
      }
    }
    __syncthreads();
    p2_last_inv<P>(rx, nv);
    p2_dc_inv<P>(rx, nv);
    __syncthreads();
    p2_pass1_inv<P>(rx, dx + e0, nv);  // g rows of this tile are already consumed
    __syncthreads();
  }
  // token split (TS > 1 threads per item, p = 256): the TS partial accumulators of an item are summed
  // in shared memory (Hx is free after the last tile) so only one thread per item issues the atomics —
  // the flush's atomics land on q^2 p addresses from every CTA (RoBERTa-base: 444 CTAs), and halving
  // them took the RoBERTa-base backward from 61.8 to 57.6 us (the whole flush cost ~5 us; r02_dd)
  if constexpr (!kAccS && TS > 1) {
    float4* red = reinterpret_cast<float4*>(Hx);  // [ts - 1][i][j][item]
    static_assert((size_t)(TS - 1) * Q * Q * NI * 16 <= (size_t)P::HF * 8, "reduction buffer fits in Hx");
    const int ts = tid / NI, item = tid % NI;
    if (ts > 0) {
#pragma unroll
      for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = 0; j < Q; ++j)
          if (i < q && j < q)
            red[(((ts - 1) * Q + i) * Q + j) * NI + item] =
                make_float4(acc[0][i][j].b1.x, acc[0][i][j].b1.y, acc[0][i][j].b2.x, acc[0][i][j].b2.y);
    }
    __syncthreads();
    if (ts > 0) return;
#pragma unroll
    for (int t2 = 1; t2 < TS; ++t2)
#pragma unroll
      for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = 0; j < Q; ++j)
          if (i < q && j < q) {
            const float4 f = red[(((t2 - 1) * Q + i) * Q + j) * NI + item];
            acc[0][i][j].b1.x += f.x;
            acc[0][i][j].b1.y += f.y;
            acc[0][i][j].b2.x += f.z;
            acc[0][i][j].b2.y += f.w;
          }
  }
#pragma unroll
  for (int a = 0; a < IPT; ++a) {
    const int u = (tid % NI) + a * NT;
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        if (i < q && j < q) {
          float* d = dw + (int64_t)(i * q + j) * N;
          BinPair v;
          if constexpr (kAccS) {
            const float4 f = *acc_slot(a, i, j);
            v = {make_float2(f.x, f.y), make_float2(f.z, f.w)};
          } else {
            v = acc[kAccS ? 0 : a][i][j];
          }
          if (u == 0) {
            atomicAdd(d + 0, v.b1.x);
            atomicAdd(d + N / 2, v.b1.y);
            atomicAdd(d + N / 4, v.b2.x);
            atomicAdd(d + 3 * N / 4, v.b2.y);
          } else {
            atomicAdd(d + u, v.b1.x);
            atomicAdd(d + N - u, v.b1.y);
            atomicAdd(d + N / 2 - u, v.b2.x);
            atomicAdd(d + N / 2 + u, v.b2.y);
          }
        }
      }
  }
}

template <typename P, int Q>
bool launch_bca_bwd3(const typename P::elem* x, const typename P::elem* w, const typename P::elem* g,
                     typename P::elem* dx, float* dw, int64_t T_, int sms, cudaStream_t st,
                     const float* wspec) {
  using L = BcaBwd3Smem<P, Q>;
  auto k = bca_bwd3_kernel<P, Q>;
  constexpr int TT = P::VT / Q;
  const int grid = bca2_grid<P>(k, P::NT, L::BYTES, (T_ + TT - 1) / TT, sms);
  if (grid <= 0) return false;
  k<<<grid, P::NT, L::BYTES, st>>>(x, w, g, dx, dw, T_, wspec);
  return true;
}

// ------------------------------------------------------------------ dispatch

template <typename P, int Q>
bool launch_bca_fwd2(const typename P::elem* x, const typename P::elem* w, typename P::elem* y, int64_t T_, int sms,
                     cudaStream_t st, int acc, const float* wspec) {
  using L = BcaFwdSmem<P, Q>;
  auto k = bca_fwd2_kernel<P, Q>;
  constexpr int TT = P::VT / Q;
  const int grid = bca2_grid<P>(k, P::NT, L::BYTES, (T_ + TT - 1) / TT, sms);
  if (grid <= 0) return false;
  k<<<grid, P::NT, L::BYTES, st>>>(x, w, y, T_, acc, wspec);
  return true;
}

template <typename P, int Q>
bool launch_bca_bwd2(const typename P::elem* x, const typename P::elem* w, const typename P::elem* g,
                     typename P::elem* dx, float* dw, int64_t T_, int sms, cudaStream_t st,
                     const float* wspec) {
  using L = BcaBwdSmem<P>;
  auto k = bca_bwd2_kernel<P, Q>;
  constexpr int TT = P::VT / Q;
  const int grid = bca2_grid<P>(k, 2 * P::NT, L::BYTES, (T_ + TT - 1) / TT, sms);
  if (grid <= 0) return false;
  k<<<grid, 2 * P::NT, L::BYTES, st>>>(x, w, g, dx, dw, T_, wspec);
  return true;
}

}  // namespace rdfft
