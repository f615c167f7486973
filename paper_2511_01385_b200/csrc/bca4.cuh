// bca4.cuh — BCA forward with independent "pipes": one CTA per SM holds the W spectra
// once (shared by all pipes) and runs PIPES thread groups, each with its own H tile and
// its own named barrier, on disjoint token tiles.  A pipe waiting at its barrier leaves
// the SM to the other pipe, so barrier and latency stalls overlap as they would across
// independent CTAs, without a second copy of W (which does not fit twice at p = 1024,
// q = 4: 72 KB each).
//
// Per tile and pipe, the same steps as bca_fwd2_kernel (Eq. 4; blocks P:L184):
//   X = rdFFT(x) (pass 1 straight from HBM) -> Y_i = sum_j W_ij (.) X_j in place ->
//   y = IrdFFT(Y) straight to HBM.  x is never written (reading C13).
#pragma once

#include "bca2.cuh"

namespace rdfft {

// bar.sync on a named barrier (ids 1..15; 0 is __syncthreads) for `nthreads` threads.
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename P, int PIPES>
struct BcaFwd4Smem {  // [H x PIPES][W][TWf][TWi]
  static constexpr int WF = kBcaQMax * kBcaQMax * P::ROWA + 16;
  static constexpr size_t H_OFF = 0;
  static constexpr size_t W_OFF = (size_t)PIPES * P::HF * 8;
  static constexpr size_t TWF_OFF = W_OFF + (size_t)WF * 8;
  static constexpr size_t TWI_OFF = TWF_OFF + (size_t)P::TWF * 8;
  static constexpr size_t BYTES = TWI_OFF + (size_t)P::TWF * 8;
};

template <typename P, int Q, int PIPES>
__global__ void __launch_bounds__(PIPES * P::NT, 1) bca_fwd4_kernel(const typename P::elem* __restrict__ x,
                                                                   const typename P::elem* __restrict__ w,
                                                                   typename P::elem* __restrict__ y, int64_t T_,
                                                                   int acc, const float* __restrict__ wspec) {
  constexpr int q = Q;
  using L = BcaFwd4Smem<P, PIPES>;
  constexpr int N = P::N, NT = P::NT;
  static_assert(Q * Q <= P::VT, "the W prologue runs on one pipe");
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  const int tid = threadIdx.x;
  const int pipe = tid / NT, lt = tid % NT;
  float2* H = reinterpret_cast<float2*>(base + L::H_OFF) + (size_t)pipe * P::HF;
  float2* Wr = reinterpret_cast<float2*>(base + L::W_OFF);
  float2* TWf = reinterpret_cast<float2*>(base + L::TWF_OFF);
  float2* TWi = reinterpret_cast<float2*>(base + L::TWI_OFF);
  const int TT = P::VT / q;  // tokens per tile
  const int64_t ntiles = (T_ + TT - 1) / TT;
  const int64_t tok_elems = (int64_t)q * N;
  p2_tables<P>(TWf, TWi, tid, PIPES * NT);
  for (int pp = 0; pp < PIPES; ++pp)
    p2_zero_pads<P>(reinterpret_cast<float2*>(base + L::H_OFF) + (size_t)pp * P::HF, P::VT, tid, PIPES * NT);
  p2_zero_pads<P>(Wr, q * q, tid, PIPES * NT);
  const uint32_t k65536 = kTwo16;
  __syncthreads();
  // ---- prologue (pipe 0): W_ij = rdFFT(w_ij) into the resident region
  if (wspec) {
    p2_load_spectra<P>(Wr, wspec, q * q, tid, PIPES * NT);
  } else if (pipe == 0) {
    const P2Roles<P> rw(Wr, TWf, TWi, lt);
    p2_pass1_fwd<P, true>(rw, w, q * q, k65536);
    named_bar(1, NT);
    p2_last_fwd<P>(rw, q * q);
    p2_dc_fwd<P>(rw, q * q);
  }
  __syncthreads();
  const P2Roles<P> rh(H, TWf, TWi, lt);
  const int bid = 1 + pipe;
  for (int64_t tile = (int64_t)blockIdx.x * PIPES + pipe; tile < ntiles; tile += (int64_t)gridDim.x * PIPES) {
    const int ntok = (int)(T_ - tile * TT < TT ? T_ - tile * TT : TT);
    const int nv = ntok * q;
    p2_pass1_fwd<P, true>(rh, x + tile * TT * tok_elems, nv, k65536);
    named_bar(bid, NT);
    p2_last_fwd<P>(rh, nv);
    p2_dc_fwd<P>(rh, nv);
    named_bar(bid, NT);
    bca_product_fwd<P, Q>(H, Wr, ntok, lt);
    named_bar(bid, NT);
    p2_last_inv<P>(rh, nv);
    p2_dc_inv<P>(rh, nv);
    named_bar(bid, NT);
    p2_pass1_inv<P>(rh, y + tile * TT * tok_elems, nv, acc != 0);
    named_bar(bid, NT);
  }
}

template <typename P, int Q, int PIPES>
bool launch_bca_fwd4(const typename P::elem* x, const typename P::elem* w, typename P::elem* y, int64_t T_, int sms,
                     cudaStream_t st, int acc, const float* wspec) {
  using L = BcaFwd4Smem<P, PIPES>;
  auto k = bca_fwd4_kernel<P, Q, PIPES>;
  constexpr int TT = P::VT / Q;
  const int grid = bca2_grid<P>(k, PIPES * P::NT, L::BYTES, ((T_ + TT - 1) / TT + PIPES - 1) / PIPES, sms);
  if (grid <= 0) return false;
  k<<<grid, PIPES * P::NT, L::BYTES, st>>>(x, w, y, T_, acc, wspec);
  return true;
}

}  // namespace rdfft
