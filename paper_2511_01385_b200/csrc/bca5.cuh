// bca5.cuh — BCA forward for the LLaMA block size (p = 1024, bf16) with the W spectra in
// TENSOR MEMORY.  The 64 KB of fp32 W spectra (q^2 <= 16 blocks) are what limit bca_fwd4 to one
// shared-memory copy and no input staging; here they live in TMEM (256 KB per SM, read with
// tcgen05.ld on a datapath separate from shared memory), which frees shared memory for a TMA
// staging buffer per pipe, so every pipe prefetches its next token tile while it computes.
//
// TMEM layout (128 columns, one allocation per CTA): the product thread of item u (bins u and
// N/2 - u, see bca2.cuh) of either pipe sits in TMEM lane u % 128 (warp w may only access lanes
// 32 (w % 4) .. + 31, and thread t of a pipe is in warp t / 32); item u's 16 bin pairs W_ij
// (4 fp32 each) are columns 64 (u / 128) .. + 63 of that lane.
//
// Per tile and pipe (Eq. 4; blocks P:L184), as bca_fwd4_kernel:
//   wait staged x tile -> X = rdFFT(x) -> issue the next tile's TMA -> Y_i = sum_j W_ij (.) X_j
//   (W from TMEM) -> y = IrdFFT(Y) straight to HBM.  x is never written (reading C13).
#pragma once

#include "bca4.cuh"

namespace rdfft {

template <typename P, int PIPES>
struct BcaFwd5Smem {  // [stage x PIPES][H x PIPES][TWf][TWi][bars x PIPES][tmem addr]
  static constexpr size_t H_OFF = (size_t)PIPES * P::STAGE;
  static constexpr size_t TWF_OFF = H_OFF + (size_t)PIPES * P::HF * 8;
  static constexpr size_t TWI_OFF = TWF_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BAR_OFF = TWI_OFF + (size_t)P::TWF * 8;
  static constexpr size_t TMEM_OFF = BAR_OFF + 8 * PIPES;
  static constexpr size_t BYTES = TMEM_OFF + 16;
};

template <typename P, int Q, int PIPES>
__global__ void __launch_bounds__(PIPES * P::NT, 1) bca_fwd5_kernel(const typename P::elem* __restrict__ x,
                                                                   const typename P::elem* __restrict__ w,
                                                                   typename P::elem* __restrict__ y, int64_t T_,
                                                                   int acc, const float* __restrict__ wspec) {
  constexpr int q = Q;
  using T = typename P::elem;
  using L = BcaFwd5Smem<P, PIPES>;
  constexpr int N = P::N, NT = P::NT, NI = N / 4, IPT = NI / NT, VT = P::VT;
  static_assert(NI == 256 && (NT == 256 || NT == 128), "one or two product items per thread, NT % 128 == 0");
  // the W prologue transforms the q*q weight rows VT at a time in the H regions of pipes 1, 2, ...
  static_assert(PIPES >= 1 + (Q * Q + VT - 1) / VT, "W prologue scratch: pipes 1.. hold q*q rows");
  constexpr uint32_t kCols = 128;
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  const int tid = threadIdx.x;
  const int pipe = tid / NT, lt = tid % NT;
  float2* Hbase = reinterpret_cast<float2*>(base + L::H_OFF);
  float2* H = Hbase + (size_t)pipe * P::HF;
  float2* TWf = reinterpret_cast<float2*>(base + L::TWF_OFF);
  float2* TWi = reinterpret_cast<float2*>(base + L::TWI_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + L::BAR_OFF) + pipe;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::TMEM_OFF);
  unsigned char* stg = base + (size_t)pipe * P::STAGE;
  const int TT = VT / q;
  const int64_t ntiles = (T_ + TT - 1) / TT;
  const int64_t tok_elems = (int64_t)q * N;
  auto tile_rows = [&](int64_t t) { return (int)((T_ - t * TT < TT ? T_ - t * TT : TT) * q); };
  if (tid < 32) {  // warp 0 owns the TMEM allocation
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  p2_tables<P>(TWf, TWi, tid, PIPES * NT);
  for (int pp = 0; pp < PIPES; ++pp) p2_zero_pads<P>(Hbase + (size_t)pp * P::HF, VT, tid, PIPES * NT);
  if (tid == 0) {
    for (int pp = 0; pp < PIPES; ++pp) mbar_init(bar - pipe + pp, 1);
    fence_mbar_init();
  }
  const uint32_t k65536 = kTwo16;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM address of item u = lt + NT m: lane u % 128 (= this thread's warp-quarter lane), 64 columns
  // per item at column 64 (u / 128)
  const uint32_t tlane = tmem + ((uint32_t)(32 * ((tid / 32) % 4)) << 16);
  auto taddr = [&](int m) { return tlane + (uint32_t)(64 * ((lt + NT * m) / 128)); };
  // ---- first tile of each pipe: start its TMA while W is being transformed
  if (lt == 0) {
    const int64_t t = (int64_t)blockIdx.x * PIPES + pipe;
    if (t < ntiles) stage_issue_rows<P>(x + t * TT * tok_elems, tile_rows(t), stg, bar);
  }
  // ---- prologue (pipe 0): W_ij = rdFFT(w_ij), VT rows at a time, into the H regions of pipes 1..
  // (scratch), then into TMEM
  if (pipe == 0) {
    for (int c0 = 0; c0 < q * q; c0 += VT) {
      float2* Wtmp = Hbase + (size_t)(1 + c0 / VT) * P::HF;
      const int nr = q * q - c0 < VT ? q * q - c0 : VT;
      if (wspec) {
        p2_load_spectra<P>(Wtmp, wspec + (int64_t)c0 * N, nr, lt, NT);
      } else {
        const P2Roles<P> rw(Wtmp, TWf, TWi, lt);
        p2_pass1_fwd<P, true>(rw, w + (int64_t)c0 * N, nr, k65536);
        named_bar(1, NT);
        p2_last_fwd<P>(rw, nr);
        p2_dc_fwd<P>(rw, nr);
      }
    }
    named_bar(1, NT);
#pragma unroll
    for (int m = 0; m < IPT; ++m) {
      const int u = lt + NT * m;
      int oa, ob;
      bca_item_offsets<P>(u, oa, ob);
#pragma unroll
      for (int g4 = 0; g4 < 4; ++g4) {  // 4 groups of 4 bin pairs = 16 columns each
        uint32_t r[16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int c = 4 * g4 + c4;
          BinPair b = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          if (c < q * q) b = bins_get(Hbase + (size_t)(1 + c / VT) * P::HF + P::row(c % VT), oa, ob, u == 0);
          r[4 * c4 + 0] = __float_as_uint(b.b1.x);
          r[4 * c4 + 1] = __float_as_uint(b.b1.y);
          r[4 * c4 + 2] = __float_as_uint(b.b2.x);
          r[4 * c4 + 3] = __float_as_uint(b.b2.y);
        }
        tmem_st16(taddr(m) + 16 * g4, r);
      }
    }
    tmem_wait_st();
  }
  tmem_fence_before();
  __syncthreads();  // W in TMEM; the scratch H regions free again (the forward never writes the pads)
  tmem_fence_after();
  const P2Roles<P> rh(H, TWf, TWi, lt);
  const int bid = 1 + pipe;
  uint32_t phase = 0;
  for (int64_t tile = (int64_t)blockIdx.x * PIPES + pipe; tile < ntiles; tile += (int64_t)gridDim.x * PIPES) {
    const int ntok = (int)(T_ - tile * TT < TT ? T_ - tile * TT : TT);
    const int nv = ntok * q;
    mbar_wait(bar, phase & 1);
    ++phase;
    p2_pass1_fwd<P>(rh, reinterpret_cast<const T*>(stg), nv, k65536);
    named_bar(bid, NT);  // H complete; staging consumed
    const int64_t nxt = tile + (int64_t)gridDim.x * PIPES;
    if (lt == 0 && nxt < ntiles) stage_issue_rows<P>(x + nxt * TT * tok_elems, tile_rows(nxt), stg, bar);
    p2_last_fwd<P>(rh, nv);
    p2_dc_fwd<P>(rh, nv);
    named_bar(bid, NT);
#pragma unroll 1
    for (int m = 0; m < IPT; ++m) {  // ---- product, W_ij from TMEM
      const int u = lt + NT * m;
      int oa, ob;
      bca_item_offsets<P>(u, oa, ob);
      const bool special = (u == 0);
      BinPair wv[Q][Q];
#pragma unroll
      for (int g4 = 0; g4 < 4; ++g4) {
        if (4 * g4 < q * q) {
          uint32_t r[16];
          tmem_ld16(taddr(m) + 16 * g4, r);
          tmem_wait_ld(r);
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int c = 4 * g4 + c4;
            if (c < q * q)
              wv[c / Q][c % Q] = {make_float2(__uint_as_float(r[4 * c4]), __uint_as_float(r[4 * c4 + 1])),
                                  make_float2(__uint_as_float(r[4 * c4 + 2]), __uint_as_float(r[4 * c4 + 3]))};
          }
        }
      }
      for (int tt = 0; tt < ntok; ++tt) {
        PrepB x1[Q];
        float2 x2[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          const BinPair xb = bins_get(H + P::row(tt * q + j), oa, ob, special);
          x1[j] = prep_b<false>(xb.b1, special);
          x2[j] = xb.b2;
        }
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          BinPair yv = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int j = 0; j < Q; ++j) {
            yv.b1 = pmac(wv[i][j].b1, x1[j], yv.b1);
            yv.b2 = cfma(wv[i][j].b2, x2[j], yv.b2);
          }
          bins_put(H + P::row(tt * q + i), oa, ob, special, yv);
        }
      }
    }
    named_bar(bid, NT);
    p2_last_inv<P>(rh, nv);
    p2_dc_inv<P>(rh, nv);
    named_bar(bid, NT);
    p2_pass1_inv<P>(rh, y + tile * TT * tok_elems, nv, acc != 0);
    named_bar(bid, NT);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols) : "memory");
}

template <typename P, int Q, int PIPES>
bool launch_bca_fwd5(const typename P::elem* x, const typename P::elem* w, typename P::elem* y, int64_t T_, int sms,
                     cudaStream_t st, int acc, const float* wspec) {
  using L = BcaFwd5Smem<P, PIPES>;
  auto k = bca_fwd5_kernel<P, Q, PIPES>;
  constexpr int TT = P::VT / Q;
  const int grid = bca2_grid<P>(k, PIPES * P::NT, L::BYTES, ((T_ + TT - 1) / TT + PIPES - 1) / PIPES, sms);
  if (grid <= 0) return false;
  k<<<grid, PIPES * P::NT, L::BYTES, st>>>(x, w, y, T_, acc, wspec);
  return true;
}

// Fused fast paths: square layers, q <= 4, p in {256, 512, 1024}.  Returns false if none applies.
template <typename T, int Q>
bool bca_fwd_fast_q(const T* x, const T* w, T* y, int64_t T_, int p, int sms, cudaStream_t st, int acc,
                    const float* wspec) {
  switch (p) {
    case 256:  // single pipe, 1-deep staging for both dtypes (bf16: the 2-pipe kernel measured
               // 0.038 -> 0.036 ms slower on RoBERTa-base, 0.048 -> 0.045 on RoBERTa-large)
      return launch_bca_fwd2<Plan2<T, 256, 16, 16, 1>, Q>(x, w, y, T_, sms, st, acc, wspec);
    case 512: return launch_bca_fwd2<Plan2<T, 512, 32, 16, 1>, Q>(x, w, y, T_, sms, st, acc, wspec);  // (2-deep / no
              // staging / 2 pipes measured equal or slower at q = 3, 4)
    // p = 2048 / 4096 (the paper's p sweep at D = 4096): the 2-pass plan with 64-point
    // register blocks (Plan2 R = 64), q * q <= VT weight spectra resident
    case 2048:
      if constexpr (Q <= 2) return launch_bca_fwd2<Plan2<T, 2048, 64, 4, 1>, Q>(x, w, y, T_, sms, st, acc, wspec);
      return false;
    case 4096:
      if constexpr (Q == 1) return launch_bca_fwd2<Plan2<T, 4096, 64, 2, 1>, Q>(x, w, y, T_, sms, st, acc, wspec);
      if constexpr (Q == 2) return launch_bca_fwd2<Plan2<T, 4096, 64, 4, 1>, Q>(x, w, y, T_, sms, st, acc, wspec);
      return false;
    case 1024:
      // bf16: W spectra in tensor memory + two staged pipes (bca_fwd5); fp32 keeps the single-pipe
      // kernel (its 8-byte direct loads made the 2-pipe variant slower: 0.194 -> 0.205 ms)
      // (four pipes of 8 vectors, two product items per thread, measured 0.141 -> 0.146 ms: slower)
      if constexpr (sizeof(T) == 2)
        return launch_bca_fwd5<Plan2<T, 1024, 32, 16>, Q, 2>(x, w, y, T_, sms, st, acc, wspec);
      else
        return launch_bca_fwd2<Plan2<T, 1024, 32, 16, 1>, Q>(x, w, y, T_, sms, st, acc, wspec);
    default: return false;
  }
}
template <typename T>
bool bca_fwd_fast(const T* x, const T* w, T* y, int64_t T_, int q_in, int q_out, int p, int sms, cudaStream_t st,
                  int acc, const float* wspec) {
  if (q_in != q_out) return false;
  switch (q_in) {
    case 1: return bca_fwd_fast_q<T, 1>(x, w, y, T_, p, sms, st, acc, wspec);
    case 2: return bca_fwd_fast_q<T, 2>(x, w, y, T_, p, sms, st, acc, wspec);
    case 3: return bca_fwd_fast_q<T, 3>(x, w, y, T_, p, sms, st, acc, wspec);
    case 4: return bca_fwd_fast_q<T, 4>(x, w, y, T_, p, sms, st, acc, wspec);
    default: return false;
  }
}

}  // namespace rdfft
