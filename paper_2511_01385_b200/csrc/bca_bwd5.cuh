// bca_bwd5.cuh — BCA backward for p = 1024 bf16 with the W spectra in TENSOR MEMORY (as
// bca_fwd5) and TMA-staged x / g tiles: the 72 KB W region of bca_bwd4 becomes two staging
// buffers, so each group prefetches its next operand tile while the CTA computes.
// Schedule, pair-split accumulators and the dx-over-g rules are bca_bwd4's (see there).
//
// TMEM (128 columns): thread t is in lane t % 128 (warp quarter rule); the four threads sharing
// a lane (t, t + 128, t + 256, t + 384) own items u = t/2 + 64 m and the same lane parity h, so
// lane L holds, at columns 32 m .. + 31, the 8 bin pairs W_ij (i = 2a + h, j = jrel(c, r)) of
// item L/2 + 64 m in the order the product reads them.
#pragma once

#include "bca_bwd4.cuh"
#include "bca5.cuh"

namespace rdfft {

template <typename P>
struct BcaBwd5Smem {  // [sx][sg][Hx][Hg][TWf][TWi][bars x 2][tmem addr]
  static constexpr size_t SG_OFF = (size_t)P::STAGE;
  static constexpr size_t HX_OFF = 2 * (size_t)P::STAGE;
  static constexpr size_t HG_OFF = HX_OFF + (size_t)P::HF * 8;
  static constexpr size_t TWF_OFF = HG_OFF + (size_t)P::HF * 8;
  static constexpr size_t TWI_OFF = TWF_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BAR_OFF = TWI_OFF + (size_t)P::TWF * 8;
  static constexpr size_t TMEM_OFF = BAR_OFF + 16;
  static constexpr size_t BYTES = TMEM_OFF + 16;
};

template <typename P, int Q>
__global__ void __launch_bounds__(2 * P::NT, 1) bca_bwd5_kernel(const typename P::elem* __restrict__ x,
                                                                const typename P::elem* __restrict__ w,
                                                                const typename P::elem* g, typename P::elem* dx,
                                                                float* __restrict__ dw, int64_t T_,
                                                                const float* __restrict__ wspec) {
  constexpr int q = Q;
  using T = typename P::elem;
  using L = BcaBwd5Smem<P>;
  constexpr int N = P::N, NT = P::NT, NT2 = 2 * NT, NI = N / 4;
  static_assert(Q * Q <= P::VT && Q % 2 == 0, "even q; the W prologue runs on one group");
  static_assert(NT2 == 2 * NI && NI == 256, "one thread pair per item, four threads per TMEM lane");
  // columns 0 .. 127: W (32 per m = t / 128); 128 .. 255: this thread's dW accumulators (32 per m)
  constexpr uint32_t kCols = 256;
  enum { kBarG0 = 1, kBarG1 = 2, kBarLI = 3 };
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float2* Hx = reinterpret_cast<float2*>(base + L::HX_OFF);
  float2* Hg = reinterpret_cast<float2*>(base + L::HG_OFF);
  float2* TWf = reinterpret_cast<float2*>(base + L::TWF_OFF);
  float2* TWi = reinterpret_cast<float2*>(base + L::TWI_OFF);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::TMEM_OFF);
  const int tid = threadIdx.x;
  const int grp = tid / NT, lt = tid % NT;
  uint64_t* gbar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF) + grp;
  unsigned char* stg = base + (grp ? L::SG_OFF : 0);
  const int TT = P::VT / q;
  const int64_t ntiles = (T_ + TT - 1) / TT;
  const int64_t tok_elems = (int64_t)q * N;
  auto tile_rows = [&](int64_t t) { return (int)((T_ - t * TT < TT ? T_ - t * TT : TT) * q); };
  const T* src = grp ? g : x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  p2_tables<P>(TWf, TWi, tid, NT2);
  p2_zero_pads<P>(Hx, P::VT, tid, NT2);
  p2_zero_pads<P>(Hg, P::VT, tid, NT2);
  if (tid == 0) {
    mbar_init(gbar, 1);
    mbar_init(gbar + 1, 1);
    fence_mbar_init();
  }
  const uint32_t k65536 = kTwo16;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (lt == 0 && (int64_t)blockIdx.x < ntiles)
    stage_issue_rows<P>(src + (int64_t)blockIdx.x * TT * tok_elems, tile_rows(blockIdx.x), stg, gbar);
  // product roles (bca_bwd4's): pair lane h owns blocks i = 2 a + h, registers relative to h
  const int u = (tid >> 1) % NI, h = tid & 1;
  int oa, ob;
  bca_item_offsets<P>(u, oa, ob);
  const bool special = (u == 0);
  constexpr int QH = Q / 2;
  auto jrel = [&](int c, int r) { return 2 * c + (r ? 1 - h : h); };
  const uint32_t taddr = tmem + ((uint32_t)(32 * ((tid / 32) % 4)) << 16) + (uint32_t)(32 * (tid / 128));
  // ---- prologue: W = rdFFT(w) into Hg (scratch) by group 0, then every thread stores its 8 pairs
  if (wspec) {
    p2_load_spectra<P>(Hg, wspec, q * q, tid, NT2);
  } else if (grp == 0) {
    const P2Roles<P> rw(Hg, TWf, TWi, lt);
    p2_pass1_fwd<P, true>(rw, w, q * q, k65536);
    named_bar(kBarG0, NT);
    p2_last_fwd<P>(rw, q * q);
    p2_dc_fwd<P>(rw, q * q);
  }
  __syncthreads();
  {
    uint32_t r16[2][16];
#pragma unroll
    for (int a = 0; a < QH; ++a)
#pragma unroll
      for (int c = 0; c < QH; ++c)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int e = (c * QH + a) * 2 + r;  // bin pair index 0 .. 2 QH^2 - 1 (<= 7): c-major
          const BinPair b = bins_get(Hg + P::row((2 * a + h) * q + jrel(c, r)), oa, ob, special);
          r16[e / 4][4 * (e % 4) + 0] = __float_as_uint(b.b1.x);
          r16[e / 4][4 * (e % 4) + 1] = __float_as_uint(b.b1.y);
          r16[e / 4][4 * (e % 4) + 2] = __float_as_uint(b.b2.x);
          r16[e / 4][4 * (e % 4) + 3] = __float_as_uint(b.b2.y);
        }
    tmem_st16(taddr, r16[0]);
    if (2 * QH * QH > 4) tmem_st16(taddr + 16, r16[1]);
    tmem_wait_st();
  }
  tmem_fence_before();
  __syncthreads();  // W in TMEM; Hg free (the forward never writes the pads)
  tmem_fence_after();
  const P2Roles<P> rm(grp ? Hg : Hx, TWf, TWi, lt);
  const P2Roles<P> rd(Hg, TWf, TWi, lt);
  // dW accumulators (2 QH^2 bin pairs per thread) live in TMEM between tiles and in registers only
  // during the product phase: held in registers across the transforms they spilled at the
  // 128-register cap.  Layout as W's (pair e = (c QH + a) 2 + r), 128 columns further.
  const uint32_t tacc = taddr + 128;
  constexpr int NACC = 2 * QH * QH;  // bin pairs (<= 8): one or two 16-column groups
  {
    uint32_t z[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) z[k] = 0u;
    tmem_st16(tacc, z);
    if (NACC > 4) tmem_st16(tacc + 16, z);
    tmem_wait_st();
  }
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int ntok = (int)(T_ - tile * TT < TT ? T_ - tile * TT : TT);
    const int nv = ntok * q;
    mbar_wait(gbar, phase & 1);
    ++phase;
    p2_pass1_fwd<P>(rm, reinterpret_cast<const T*>(stg), nv, k65536);
    named_bar(grp ? kBarG1 : kBarG0, NT);  // this group's staging buffer consumed
    const int64_t nxt = tile + gridDim.x;
    if (lt == 0 && nxt < ntiles) stage_issue_rows<P>(src + nxt * TT * tok_elems, tile_rows(nxt), stg, gbar);
    p2_last_fwd<P>(rm, nv);
    p2_dc_fwd<P>(rm, nv);
    __syncthreads();
    // ---- products (W from TMEM, c-major layout: the 2 QH bin pairs of input-block pair c are one
    // 16-column group, loaded per (token, c), so only a quarter of W is live in registers at a time;
    // holding all of W across the token loop spilled 20 B at the 128-register cap)
    BinPair acc[QH][QH][2];
    {
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
            const int e = (c * QH + a) * 2 + r;
            const uint32_t* f = &r16[e / 4][4 * (e % 4)];
            acc[a][c][r] = {make_float2(__uint_as_float(f[0]), __uint_as_float(f[1])),
                            make_float2(__uint_as_float(f[2]), __uint_as_float(f[3]))};
          }
    }
    for (int tt = 0; tt < ntok; ++tt) {
      float2 g2[QH];
      PrepB g1[QH];
#pragma unroll
      for (int a = 0; a < QH; ++a) {
        const BinPair gb = bins_get(Hg + P::row(tt * q + 2 * a + h), oa, ob, special);
        g1[a] = prep_b<true>(gb.b1, special);
        g2[a] = gb.b2;
      }
#pragma unroll
      for (int c = 0; c < QH; ++c) {
        BinPair wv[QH][2];
        {
          uint32_t r16[16];
          tmem_ld16(taddr + 16 * (2 * QH * c / 4), r16);
          tmem_wait_ld(r16);
#pragma unroll
          for (int a = 0; a < QH; ++a)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const int e = (2 * QH * c + 2 * a + r) % 4;  // position inside the 4-pair group
              wv[a][r] = {make_float2(__uint_as_float(r16[4 * e]), __uint_as_float(r16[4 * e + 1])),
                          make_float2(__uint_as_float(r16[4 * e + 2]), __uint_as_float(r16[4 * e + 3]))};
            }
        }
        BinPair xv[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) xv[r] = bins_get(Hx + P::row(tt * q + jrel(c, r)), oa, ob, special);
        BinPair d[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          d[r] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int a = 0; a < QH; ++a) {
            acc[a][c][r].b1 = pmac(xv[r].b1, g1[a], acc[a][c][r].b1);
            acc[a][c][r].b2 = cfmac(xv[r].b2, g2[a], acc[a][c][r].b2);
            d[r].b1 = pmac(wv[a][r].b1, g1[a], d[r].b1);
            d[r].b2 = cfmac(wv[a][r].b2, g2[a], d[r].b2);
          }
        }
        d[0].b1.x += __shfl_xor_sync(0xffffffffu, d[1].b1.x, 1);
        d[0].b1.y += __shfl_xor_sync(0xffffffffu, d[1].b1.y, 1);
        d[0].b2.x += __shfl_xor_sync(0xffffffffu, d[1].b2.x, 1);
        d[0].b2.y += __shfl_xor_sync(0xffffffffu, d[1].b2.y, 1);
        bins_put(Hg + P::row(tt * q + jrel(c, 0)), oa, ob, special, d[0]);
      }
    }
    {
      uint32_t r16[2][16];
#pragma unroll
      for (int a = 0; a < QH; ++a)
#pragma unroll
        for (int c = 0; c < QH; ++c)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int e = (c * QH + a) * 2 + r;
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
  uint32_t fin[2][16];
  tmem_ld16(tacc, fin[0]);
  if (NACC > 4) tmem_ld16(tacc + 16, fin[1]);
  tmem_wait_ld(fin[0]);
  if (NACC > 4) tmem_wait_ld(fin[1]);
  // ---- flush dW accumulators into dw (packed slots) with fp32 atomics
#pragma unroll
  for (int a = 0; a < QH; ++a)
#pragma unroll
    for (int c = 0; c < QH; ++c)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = 2 * a + h, j = jrel(c, r);
        float* d = dw + (int64_t)(i * q + j) * N;
        const int e = (c * QH + a) * 2 + r;
        const uint32_t* f = &fin[e / 4][4 * (e % 4)];
        const BinPair v = {make_float2(__uint_as_float(f[0]), __uint_as_float(f[1])),
                           make_float2(__uint_as_float(f[2]), __uint_as_float(f[3]))};
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
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols) : "memory");
}

template <typename P, int Q>
bool launch_bca_bwd5(const typename P::elem* x, const typename P::elem* w, const typename P::elem* g,
                     typename P::elem* dx, float* dw, int64_t T_, int sms, cudaStream_t st,
                     const float* wspec) {
  using L = BcaBwd5Smem<P>;
  auto k = bca_bwd5_kernel<P, Q>;
  constexpr int TT = P::VT / Q;
  const int grid = bca2_grid<P>(k, 2 * P::NT, L::BYTES, (T_ + TT - 1) / TT, sms);
  if (grid <= 0) return false;
  k<<<grid, 2 * P::NT, L::BYTES, st>>>(x, w, g, dx, dw, T_, wspec);
  return true;
}

// Measured (B200, T = 16384, bf16): LLaMA shape (p = 1024, q = 4) bwd4 0.319 -> 0.300 ms over bwd2 and
// bwd5 (W in TMEM) 0.276 ms; RoBERTa-large (p = 256, q = 4) 0.110 -> 0.097 ms; p = 256 runs bwd3.
// The pair-split kernel (bwd4) only for even q (odd q: half the pair-split product is predicated off).
template <typename T, int Q>
bool bca_bwd_fast_q(const T* x, const T* w, const T* g, T* dx, float* dw, int64_t T_, int p, int sms,
                    cudaStream_t st, const float* wspec) {
  switch (p) {
    case 256:  // the single-group kernel (all threads in every phase): RoBERTa-base bf16 bwd 0.073 -> 0.061 ms,
               // RoBERTa-large 0.098 -> 0.081 ms (the 2-group / pair-split kernels measured slower here)
      return launch_bca_bwd3<Plan2<T, 256, 16, 16>, Q>(x, w, g, dx, dw, T_, sms, st, wspec);
    case 512:  // (the single-group kernel measured slower here: 0.171 -> 0.200 ms at q = 4)
      if constexpr (Q % 2 == 0) return launch_bca_bwd4<Plan2<T, 512, 32, 16>, Q>(x, w, g, dx, dw, T_, sms, st, wspec);
      else return launch_bca_bwd2<Plan2<T, 512, 32, 8>, Q>(x, w, g, dx, dw, T_, sms, st, wspec);
    case 1024:
      if constexpr (sizeof(T) == 2 && Q % 2 == 0)
        return launch_bca_bwd5<Plan2<T, 1024, 32, 16>, Q>(x, w, g, dx, dw, T_, sms, st, wspec);
      else if constexpr (Q % 2 == 0)
        return launch_bca_bwd4<Plan2<T, 1024, 32, 16>, Q>(x, w, g, dx, dw, T_, sms, st, wspec);
      else
        return launch_bca_bwd3<Plan2<T, 1024, 32, 16>, Q>(x, w, g, dx, dw, T_, sms, st, wspec);
    case 2048:  // see bca_fwd_fast_q
      if constexpr (Q <= 2) return launch_bca_bwd3<Plan2<T, 2048, 64, 4>, Q>(x, w, g, dx, dw, T_, sms, st, wspec);
      return false;
    case 4096:
      if constexpr (Q == 1) return launch_bca_bwd3<Plan2<T, 4096, 64, 4>, Q>(x, w, g, dx, dw, T_, sms, st, wspec);
      return false;
    default: return false;
  }
}

template <typename T>
bool bca_bwd_fast(const T* x, const T* w, const T* g, T* dx, float* dw, int64_t T_, int q_in, int q_out, int p,
                  int sms, cudaStream_t st, const float* wspec) {
  if (q_in != q_out) return false;
  switch (q_in) {
    case 1: return bca_bwd_fast_q<T, 1>(x, w, g, dx, dw, T_, p, sms, st, wspec);
    case 2: return bca_bwd_fast_q<T, 2>(x, w, g, dx, dw, T_, p, sms, st, wspec);
    case 3: return bca_bwd_fast_q<T, 3>(x, w, g, dx, dw, T_, p, sms, st, wspec);
    case 4: return bca_bwd_fast_q<T, 4>(x, w, g, dx, dw, T_, p, sms, st, wspec);
    default: return false;
  }
}

}  // namespace rdfft
