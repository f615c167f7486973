// bca_bwd4.cuh — BCA backward (Eq. 5; block pairing C11) with two overlapped
// thread groups and pair-split dW accumulators.
//
// 2 NT threads per CTA (one CTA per SM; W spectra resident in shared memory, as in bca2.cuh).
// Group 0 transforms x, group 1 transforms g; the product runs on all threads; then the two
// groups split the inverse and overlap it with the next tile:
//
//   g0: P1X(t) LX(t) | PR(t) | LI(t) -> arrive | P1X(t+1) LX(t+1) | PR(t+1) ...
//   g1: P1G(t) LG(t) | PR(t) | wait LI(t) P1I(t) | P1G(t+1) LG(t+1) | PR(t+1) ...
//
// (P1 = pass 1, L = last pass, PR = product, LI / P1I = inverse last pass / pass 1.)
// Product: thread pair (2u, 2u+1) owns item u (bins u and N/2-u, see bca2.cuh); lane h of
// the pair owns the output blocks i with i % 2 == h:
//   Acc_ij += conj(X_j) (.) G_i  for its i, every j   (fp32 registers for the whole token range)
//   d_j = sum_{its i} conj(W_ij) (.) G_i; the pair exchanges halves with one shuffle per value,
//   and lane h writes D_j = d_j + d'_j for j % 2 == h over G_j (rows it alone read), so the
//   inverse runs on Hg and Hx is free for the next tile as soon as the product ends.
// dx may alias g: tile t's g rows are read (P1G(t)) before its dx rows are written
// (P1I(t)), and no other tile touches those rows.
#pragma once

#include "bca4.cuh"

namespace rdfft {

// bar.arrive on a named barrier: signal without waiting (producer side of a bar.sync).
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename P, int Q>
__global__ void __launch_bounds__(2 * P::NT, 1) bca_bwd4_kernel(const typename P::elem* __restrict__ x,
                                                                const typename P::elem* __restrict__ w,
                                                                const typename P::elem* g, typename P::elem* dx,
                                                                float* __restrict__ dw, int64_t T_,
                                                                const float* __restrict__ wspec) {
  constexpr int q = Q;
  using T = typename P::elem;
  using L = BcaBwd3Smem<P>;
  constexpr int N = P::N, NT = P::NT, NT2 = 2 * NT, NI = N / 4;
  static_assert(Q * Q <= P::VT, "the W prologue runs on one group");
  static_assert(NT2 % (2 * NI) == 0, "thread pairs cover the items");
  constexpr int TS = NT2 / (2 * NI);  // token split of the product
  enum { kBarG0 = 1, kBarG1 = 2, kBarLI = 3 };
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float2* Hx = reinterpret_cast<float2*>(base + L::HX_OFF);
  float2* Hg = reinterpret_cast<float2*>(base + L::HG_OFF);
  float2* Wr = reinterpret_cast<float2*>(base + L::W_OFF);
  float2* TWf = reinterpret_cast<float2*>(base + L::TWF_OFF);
  float2* TWi = reinterpret_cast<float2*>(base + L::TWI_OFF);
  const int tid = threadIdx.x;
  const int grp = tid / NT, lt = tid % NT;
  const int TT = P::VT / q;
  const int64_t ntiles = (T_ + TT - 1) / TT;
  const int64_t tok_elems = (int64_t)q * N;
  p2_tables<P>(TWf, TWi, tid, NT2);
  p2_zero_pads<P>(Hx, P::VT, tid, NT2);
  p2_zero_pads<P>(Hg, P::VT, tid, NT2);
  p2_zero_pads<P>(Wr, q * q, tid, NT2);
  const uint32_t k65536 = kTwo16;
  // dW accumulators in TMEM between tiles (in registers only during the product phase; held across
  // the transforms they spilled at the 128-register cap): thread t owns lane t % 128, columns
  // 32 (t / 128) .. + 31, bin pair e = (a QH + c) 2 + r at columns 4 e .. 4 e + 3
  constexpr uint32_t kCols = 128;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::TMEM_OFF);
  tmem_alloc<kCols>(tmem_slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tacc = tmem + ((uint32_t)(32 * ((tid / 32) % 4)) << 16) + (uint32_t)(32 * (tid / 128));
  if (wspec) {
    p2_load_spectra<P>(Wr, wspec, q * q, tid, NT2);
  } else if (grp == 0) {  // W_ij = rdFFT(w_ij), q*q <= VT vectors
    const P2Roles<P> rw(Wr, TWf, TWi, lt);
    p2_pass1_fwd<P, true>(rw, w, q * q, k65536);
    named_bar(kBarG0, NT);
    p2_last_fwd<P>(rw, q * q);
    p2_dc_fwd<P>(rw, q * q);
  }
  __syncthreads();
  const P2Roles<P> rm(grp ? Hg : Hx, TWf, TWi, lt);  // this group's forward operand
  const P2Roles<P> rd(Hg, TWf, TWi, lt);              // D (inverse) lives in Hg
  const T* src = grp ? g : x;
  // product roles: pair lane h owns blocks i = 2 a + h; its registers index the input blocks
  // relative to h, j(c, r) = 2 c + (r ? 1 - h : h): r = 0 is the D_j it writes, r = 1 the one
  // it hands to its partner (no per-lane register selects).
  const int u = (tid >> 1) % NI, h = tid & 1, ts = (tid >> 1) / NI;
  int oa, ob;
  bca_item_offsets<P>(u, oa, ob);
  const bool special = (u == 0);
  constexpr int QH = (Q + 1) / 2;
  auto jrel = [&](int c, int r) { return 2 * c + (r ? 1 - h : h); };
  constexpr int NACC = 2 * QH * QH;  // bin pairs per thread (<= 8): one or two 16-column groups
  {
    uint32_t z[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) z[k] = 0u;
    tmem_st16(tacc, z);
    if (NACC > 4) tmem_st16(tacc + 16, z);
    tmem_wait_st();
  }
  auto acc_load = [&](BinPair (&acc)[QH][QH][2]) {
    uint32_t r16[2][16];
    tmem_ld16(tacc, r16[0]);
    if (NACC > 4) tmem_ld16(tacc + 16, r16[1]);
    tmem_wait_ld(r16[0]);
    if (NACC > 4) tmem_wait_ld(r16[1]);
#pragma unroll
    for (int a = 0; a < QH; ++a)
#pragma unroll
      for (int c = 0; c < QH; ++c)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int e = (a * QH + c) * 2 + r;
          const uint32_t* f = &r16[e / 4][4 * (e % 4)];
          acc[a][c][r] = {make_float2(__uint_as_float(f[0]), __uint_as_float(f[1])),
                          make_float2(__uint_as_float(f[2]), __uint_as_float(f[3]))};
        }
  };
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int ntok = (int)(T_ - tile * TT < TT ? T_ - tile * TT : TT);
    const int nv = ntok * q;
    // ---- forward transforms of this group's operand
    p2_pass1_fwd<P, true>(rm, src + tile * TT * tok_elems, nv, k65536);
    named_bar(grp ? kBarG1 : kBarG0, NT);
    p2_last_fwd<P>(rm, nv);
    p2_dc_fwd<P>(rm, nv);
    __syncthreads();
    // ---- products
    {
      BinPair acc[QH][QH][2];
      acc_load(acc);
      BinPair wv[QH][QH][2];
#pragma unroll
      for (int a = 0; a < QH; ++a)
#pragma unroll
        for (int c = 0; c < QH; ++c)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int i = 2 * a + h, j = jrel(c, r);
            if (i < q && j < q) wv[a][c][r] = bins_get(Wr + P::row(i * q + j), oa, ob, special);
          }
      for (int tt = ts; tt < ntok; tt += TS) {
        BinPair xv[QH][2];
        float2 g2[QH];
        PrepB g1[QH];
#pragma unroll
        for (int c = 0; c < QH; ++c)
#pragma unroll
          for (int r = 0; r < 2; ++r)
            if (jrel(c, r) < q) xv[c][r] = bins_get(Hx + P::row(tt * q + jrel(c, r)), oa, ob, special);
#pragma unroll
        for (int a = 0; a < QH; ++a)
          if (2 * a + h < q) {
            const BinPair gb = bins_get(Hg + P::row(tt * q + 2 * a + h), oa, ob, special);
            g1[a] = prep_b<true>(gb.b1, special);
            g2[a] = gb.b2;
          }
#pragma unroll
        for (int c = 0; c < QH; ++c) {
          BinPair d[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            d[r] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int a = 0; a < QH; ++a)
              if (2 * a + h < q && jrel(c, r) < q) {
                acc[a][c][r].b1 = pmac(xv[c][r].b1, g1[a], acc[a][c][r].b1);
                acc[a][c][r].b2 = cfmac(xv[c][r].b2, g2[a], acc[a][c][r].b2);
                d[r].b1 = pmac(wv[a][c][r].b1, g1[a], d[r].b1);
                d[r].b2 = cfmac(wv[a][c][r].b2, g2[a], d[r].b2);
              }
          }
          // lane h keeps D_{2c+h} and receives its partner's partial of the same block
          d[0].b1.x += __shfl_xor_sync(0xffffffffu, d[1].b1.x, 1);
          d[0].b1.y += __shfl_xor_sync(0xffffffffu, d[1].b1.y, 1);
          d[0].b2.x += __shfl_xor_sync(0xffffffffu, d[1].b2.x, 1);
          d[0].b2.y += __shfl_xor_sync(0xffffffffu, d[1].b2.y, 1);
          if (jrel(c, 0) < q) bins_put(Hg + P::row(tt * q + jrel(c, 0)), oa, ob, special, d[0]);
        }
      }
      uint32_t r16[2][16];
#pragma unroll
      for (int a = 0; a < QH; ++a)
#pragma unroll
        for (int c = 0; c < QH; ++c)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int e = (a * QH + c) * 2 + r;
            uint32_t* f = &r16[e / 4][4 * (e % 4)];
            f[0] = __float_as_uint(acc[a][c][r].b1.x);
            f[1] = __float_as_uint(acc[a][c][r].b1.y);
            f[2] = __float_as_uint(acc[a][c][r].b2.x);
            f[3] = __float_as_uint(acc[a][c][r].b2.y);
          }
      tmem_st16(tacc, r16[0]);
      if (NACC > 4) tmem_st16(tacc + 16, r16[1]);
      tmem_wait_st();
    }
    __syncthreads();  // D complete in Hg; Hx free
    if (grp == 0) {
      p2_last_inv<P>(rd, nv);
      p2_dc_inv<P>(rd, nv);
      named_arrive(kBarLI, NT2);
    } else {
      named_bar(kBarLI, NT2);
      p2_pass1_inv<P>(rd, dx + tile * TT * tok_elems, nv);
      named_bar(kBarG1, NT);  // Hg free for the next tile's g
    }
  }
  // ---- flush dW accumulators into dw (packed slots) with fp32 atomics
  BinPair acc[QH][QH][2];
  acc_load(acc);
#pragma unroll
  for (int a = 0; a < QH; ++a)
#pragma unroll
    for (int c = 0; c < QH; ++c)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
      const int i = 2 * a + h, j = jrel(c, r);
      if (i < q && j < q) {
        float* d = dw + (int64_t)(i * q + j) * N;
        const BinPair v = acc[a][c][r];
        if (special) {
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
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  tmem_free<kCols>(tmem);
}

template <typename P, int Q>
bool launch_bca_bwd4(const typename P::elem* x, const typename P::elem* w, const typename P::elem* g,
                     typename P::elem* dx, float* dw, int64_t T_, int sms, cudaStream_t st,
                     const float* wspec) {
  using L = BcaBwd3Smem<P>;
  auto k = bca_bwd4_kernel<P, Q>;
  constexpr int TT = P::VT / Q;
  const int grid = bca2_grid<P>(k, 2 * P::NT, L::BYTES, (T_ + TT - 1) / TT, sms);
  if (grid <= 0) return false;
  k<<<grid, 2 * P::NT, L::BYTES, st>>>(x, w, g, dx, dw, T_, wspec);
  return true;
}

}  // namespace rdfft
