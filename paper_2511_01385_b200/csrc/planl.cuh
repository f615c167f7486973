// planl.cuh — in-place rdFFT for large n (8192, 16384, 32768), one vector
// per CTA held in shared memory as fp32 (<= 128 KB), three register passes.
//
// n = 32 * 32 * M3 (M3 = n / 1024 in {8, 16, 32}); every pass is the paper's radix-2 stages
// (Prop. 1) regrouped on the closed sets of SURVEY §0 fact 4:
//   pass 1 (stages m = 1 .. 16): the 32-point packed real FFT of each decimated subsequence
//           x[r :: n/32] (bit reversal absorbed: subsequence r lands in window rev(r));
//   pass 2 (stages m = 32 .. 512) on each 1024-slot window: S_k = {32 j + k, 32 (j+1) - k},
//           k = 1 .. 15 -> twiddle W_1024^{k rev(j)} + 32-point complex DIT; k = 16 (block
//           Nyquists) the same with zero imaginary input; k = 0 (block DCs) a real 32-point FFT;
//   pass 3 (stages m = 1024 .. n/2) on the whole vector: S_k = {1024 j +- k}, k = 1 .. 512,
//           twiddle W_n^{k rev(j)} + M3-point DIT; k = 0 a real M3-point FFT.
// The inverse runs the reversed graph (Eq. 7): pass 3, 2, 1 with conjugate
// twiddles, unscaled, 1/n folded into pass 3 (reading C4).
//
// Shared layout: plain packed slots (fp32), 32-slot windows, 16-byte chunks XOR-swizzled by
// window bits so the pass-1 window stores and the pass-2/3 set accesses are conflict-free
// (simulated: <= 1.5 wavefronts per ideal one).  Twiddle tables in shared memory:
// TW2[j][k-1] = W_1024^{k rev5(j)} (4 KB) and TW3[a][k-1] = W_n^{4 k a} (M3/4 x 512) with
// W_n^{k b}, b < 4, in registers.  No global scratch.
//
// n = 65536 (NC = 2): a thread-block cluster of two CTAs (one per SM, DSMEM between them).  By the
// per-stage invariant (DIT), after log2(n/2) stages window r in {0, 1} of the vector holds the
// packed n/2-point spectrum of x[r :: 2], so CTA r runs the n/2 = 32768 plan above on x[r :: 2]
// (strided loads) into its own shared memory; the last stage (m = n/2, beta = 0: Prop. 1's groups
// {k, m - k, m + k, 2m - k}) reads one half pair from each CTA (the peer's through
// ld.shared::cluster) and stores the four outputs straight to HBM.  The inverse runs Eq. 7's first
// stage (m = n/2, with its 1/2) from HBM into both CTAs' shared memory (the peer's half through
// st.shared::cluster), then each CTA the exact n/2-point inverse with strided stores.
#pragma once

#include <cooperative_groups.h>

#include "plan2.cuh"

namespace rdfft {

template <typename T, int N_>
struct PlanL {
  using elem = T;
  static constexpr int N = N_, LN = ilog2c<N>();
  static constexpr int R = 32, LR = 5, S = N / R, LS = LN - LR;
  static constexpr int M2 = 32, W2 = 1024, NW2 = N / W2;
  static constexpr int M3 = N / W2, LM3 = ilog2c<M3>(), K3 = W2 / 2;
  // threads: one per pass-1 subsequence pair and per pass-2 set (S/2 = 16 NW2), <= 16 warps (4 per
  // SM quadrant keeps the 128-register budget); pass 3 loops over K3 / NT sets per thread.  Small n
  // thus runs several CTAs per SM (n = 8192: 128 threads, 4 CTAs; 16384: 256 threads, 2 CTAs).
  static constexpr int NT = S / 2 < 512 ? S / 2 : 512;
  static constexpr int K3PT = K3 / NT;
  static constexpr int MINB = 512 / NT;  // CTAs per SM the 128-register budget allows
  static_assert(S / 2 == NW2 * 16 || NT == 512, "pass-2 sets per thread");
  // TW2: 32 x 17 pass-2 twiddles, then W_32^t (t < 16) for the warp-cooperative pass-3 DC set (dc_warp_dit)
  static constexpr int TW2N = 32 * 17 + 16, TW3N = (M3 / 4) * K3;
  static constexpr int HPAD = 64;  // additive pad: 4 floats per n/16 slots (see phys)
  static constexpr size_t TW2_OFF = (size_t)(N + HPAD) * 4;
  static constexpr size_t TW3_OFF = TW2_OFF + (size_t)TW2N * 8;
  static constexpr size_t BYTES1 = TW3_OFF + (size_t)TW3N * 8;
  // cluster pair (n = 2N): cross-stage twiddles W_{2N}^{128 a} (a < N / 256) and W_{2N}^b (b < 128)
  static constexpr int TWCA = N / 256, TWCB = 128;
  static constexpr size_t TWC_OFF = BYTES1;
  static constexpr size_t BYTES2 = TWC_OFF + (size_t)(TWCA + TWCB) * 8;
  // kST (one-CTA plan, one pass-3 set per thread: n = 32768): pass 3's natural-order side is a row
  // staged in shared memory at H's start (it aliases H: a barrier separates pass 3's reads of H from its
  // writes) — the forward's outputs leave through TMA bulk stores, the inverse's inputs arrive by a TMA
  // bulk load issued as soon as the previous vector's pass 1 has read H — instead of one 2-byte
  // global access per slot (lg_throttle-bound at one CTA per SM).  mbarrier at BAR_OFF.
  static constexpr bool kST = (K3PT * M3 <= 32);  // all of a thread's pass-3 sets fit in 64 registers
  static constexpr size_t BAR_OFF = BYTES1;
  static constexpr size_t BYTES = BYTES1 + 16;
  static_assert((size_t)N * sizeof(T) <= (size_t)N * 4, "the staged row fits in H");
  static_assert(!kST || S / 2 == NT, "kST: every thread runs pass 1 (barriers inside it)");
  static_assert(M3 >= 8 && M3 <= 32 && LS >= 8, "plan L shape");
  static_assert(4 * NT == (N >> 4), "store/load phase chunk i sits in pad period i");
  static_assert(NW2 % (2 * (N / 4096)) == 0, "pass-2 half-warp block pairing");
  // Float index of packed slot s: plain slots plus 4 floats of pad per n/16 slots.  The pass-1
  // float4 window stores of 8 consecutive lanes differ exactly in slot bits LN-4 .. LN-2 (the
  // bit-reversed low bits of their subsequence index), so the pad puts them on 8 distinct 16-byte
  // bank groups; and since the pad only changes at multiples of n/16 >= 512 slots, every pass-2/3
  // access is a per-thread base plus a compile-time offset (OffP2 / OffP3), no runtime arithmetic.
  __host__ __device__ static constexpr int pad(int s) { return 4 * (s >> (LN - 4)); }
  __host__ __device__ static constexpr int phys(int s) { return s + pad(s); }
};

// Compile-time offsets of a closed set's two slots {be + j m0 + k, be + (j+1) m0 - k} relative to
// per-thread bases pa = &H[phys(be) + k] and pb = &H[phys(be) - k] (valid for 1 <= k <= m0/2 and
// be a multiple of the pad period or of m0 * M; see PlanL::phys).
template <typename P>
struct OffP3 {  // pass 3: be = 0, m0 = 1024, k < 512 (k = 512: the half set uses b() for both)
  __host__ __device__ static constexpr int a(int j) { return 1024 * j + P::pad(1024 * j); }
  __host__ __device__ static constexpr int b(int j) { return 1024 * (j + 1) + P::pad(1024 * (j + 1) - 1); }
};
template <typename P>
struct OffP2 {  // pass 2: be = ww 1024, m0 = 32, k <= 16; in-block pad only when n/16 < 1024
  __host__ __device__ static constexpr int rel(int x) { return (P::LN - 4 < 10) ? 4 * (x >> (P::LN - 4)) : 0; }
  __host__ __device__ static constexpr int a(int j) { return 32 * j + rel(32 * j); }
  __host__ __device__ static constexpr int b(int j) { return 32 * (j + 1) + rel(32 * j + 31); }
};

// pass-3 twiddle W_n^{k r} for compile-time r = 4 a + b
template <int K3>
struct LTw3 {
  const float2* h;  // &TW3[0][k-1]
  float2 w1, w2, w3;
  template <int R_>
  __device__ __forceinline__ float2 at() const {
    constexpr int a = R_ >> 2, b = R_ & 3;
    const float2 t = h[a * K3];
    if constexpr (b == 0) return t;
    const float2 w = b == 1 ? w1 : (b == 2 ? w2 : w3);
    return make_float2(fmaf(t.x, w.x, -t.y * w.y), fmaf(t.x, w.y, t.y * w.x));
  }
};

// One closed set of a pass: M blocks of size m0, set k (1 <= k <= m0/2), slots pa[OFF::a(j)]
// (= be + j m0 + k) and pb[OFF::b(j)] (= be + (j+1) m0 - k).  half (k == m0/2, the zero-imaginary
// set): both are the same slot; kHalfB: read it through pb (the pass-3 half set, whose pad follows
// b()).  tw.template at<r>() = W_W^{k r} (forward) / conj (inverse).
// kG (pass 3 of the one-CTA plan): the forward stores its outputs to a natural-order row and the
// inverse reads its inputs from one — slot be + j m0 + k at ga[j m0], slot be + (j+1) m0 - k at
// gb[(j+1) m0] (ga = row + k, gb = row - k) — instead of H: the global row itself (ST = gio<T>,
// LD = gio1<T>) or the staged row in shared memory (ST = sst1<T>, LD = sio1<T>; PlanL::kST).
// Split in two phases so the staged pass 3 can put a barrier between them: pl_set_in reads the set
// and runs its arithmetic into (zr, zi), pl_set_out writes the results.
struct NoFix {
  template <int M>
  __device__ __forceinline__ void operator()(float (&)[M], float (&)[M]) const {}
};

// fix(zr, zi) runs right after the loads (before the forward's twiddles / the inverse's DIT): pass 2's
// paired block-DC / block-Nyquist sets (PairFix below) hook in there.
template <typename P, int M, bool kInv, typename OFF, bool kHalfB = false, bool kG = false,
          typename LD = gio1<typename P::elem>, typename TW, typename FIX = NoFix>
__device__ __forceinline__ void pl_set_in(float (&zr)[M], float (&zi)[M], float* pa, float* pb, bool half,
                                          const TW& tw, const typename P::elem* ga = nullptr,
                                          const typename P::elem* gb = nullptr, int m0 = 0, uint32_t k65536 = 0,
                                          const FIX& fix = FIX{}) {
  constexpr int LM = ilog2c<M>();
  auto A = [&](auto J) -> float& {
    constexpr int j = decltype(J)::value;
    if constexpr (kHalfB) return pb[OFF::b(j)];
    else return pa[OFF::a(j)];
  };
  auto B = [&](auto J) -> float& {
    constexpr int j = decltype(J)::value;
    return pb[OFF::b(j)];
  };
  if (!kInv) {
    ct::static_for<0, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      zr[j] = A(J);
      if constexpr (kHalfB) zi[j] = 0.f;
      else zi[j] = half ? 0.f : B(J);
    });
    fix(zr, zi);
    ct::static_for<1, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 t = tw.template at<rev_bits<LM>(j)>();
      const float q = zr[j];
      zr[j] = fmaf(q, t.x, -zi[j] * t.y);
      zi[j] = fmaf(q, t.y, zi[j] * t.x);
    });
    cfft_dit<M>(zr, zi);
  } else {
    // Y[q] into register rev(q): q < M/2: Re at A(q), Im at B(M-1-q); q >= M/2: Re at B(M-1-q),
    // Im = -(value at A(q)).  Half set: A(q) = B(q) real for q < M/2 (mirror of the forward).
    ct::static_for<0, M>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int rq = rev_bits<LM>(q);
      if constexpr (kG) {
        const float av = LD::ld(ga + q * m0, k65536), bv = LD::ld(gb + (M - q) * m0, k65536);
        if constexpr (q < M / 2) {
          zr[rq] = av;
          zi[rq] = bv;
        } else {
          zr[rq] = bv;
          zi[rq] = -av;
        }
      } else if constexpr (kHalfB) {
        if constexpr (q < M / 2) {
          zr[rq] = A(Q);
          zi[rq] = B(ct::ic<M - 1 - q>{});
        } else {
          zr[rq] = B(ct::ic<M - 1 - q>{});
          zi[rq] = -A(Q);
        }
      } else {
        const float av = A(Q), bv = B(ct::ic<M - 1 - q>{});
        if constexpr (q < M / 2) {
          zr[rq] = av;
          zi[rq] = bv;
        } else {
          zr[rq] = bv;
          zi[rq] = -av;
        }
      }
    });
    fix(zr, zi);
    cfft_dit<M, true>(zr, zi);
    ct::static_for<0, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      constexpr int rj = rev_bits<LM>(j);
      const float2 t = tw.template at<rj>();
      const float q = zr[rj];
      zr[rj] = fmaf(q, t.x, -zi[rj] * t.y);
      zi[rj] = fmaf(q, t.y, zi[rj] * t.x);
    });
  }
}

// skipB0 (forward, H side): leave out the B stores of q = 0 and q = M/2 — pass 2's paired DC sets, whose
// window-2 store base is shifted by one block (pair_dc_fwd_inplace): q = 0 would leave the window and
// q = M/2 (slot 32 * 16) would take the pad offset of the block before it; the caller stores those two.
template <typename P, int M, bool kInv, typename OFF, bool kHalfB = false, bool kG = false,
          typename ST = gio<typename P::elem>>
__device__ __forceinline__ void pl_set_out(const float (&zr)[M], const float (&zi)[M], float* pa, float* pb,
                                           bool half, typename P::elem* ga = nullptr, typename P::elem* gb = nullptr,
                                           int m0 = 0, bool skipB0 = false) {
  constexpr int LM = ilog2c<M>();
  auto A = [&](auto J) -> float& {
    constexpr int j = decltype(J)::value;
    if constexpr (kHalfB) return pb[OFF::b(j)];
    else return pa[OFF::a(j)];
  };
  auto B = [&](auto J) -> float& {
    constexpr int j = decltype(J)::value;
    return pb[OFF::b(j)];
  };
  if (!kInv) {
    // slot be + q m0 + k <- (q < M/2 ? Re : -Im) Y[q];  be + (M - q) m0 - k (= B(M-1-q)) <- the other
    ct::static_for<0, M>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      if constexpr (kG) {
        if constexpr (q < M / 2) {
          ST::st1(ga + q * m0, zr[q]);
          ST::st1(gb + (M - q) * m0, zi[q]);
        } else if constexpr (!kHalfB) {
          if (!half) {
            ST::st1(ga + q * m0, -zi[q]);
            ST::st1(gb + (M - q) * m0, zr[q]);
          }
        }
      } else if constexpr (q < M / 2) {  // (half set: B(M-1-q) is another slot of the same set)
        A(Q) = zr[q];
        if (q != 0 || !skipB0) B(ct::ic<M - 1 - q>{}) = zi[q];
      } else if constexpr (!kHalfB) {
        if (!half) {
          A(Q) = -zi[q];
          if (q != M / 2 || !skipB0) B(ct::ic<M - 1 - q>{}) = zr[q];
        }
      }
    });
  } else {
    ct::static_for<0, M>([&](auto J) {
      constexpr int j = decltype(J)::value;
      constexpr int rj = rev_bits<LM>(j);
      A(J) = zr[rj];
      if constexpr (!kHalfB) {
        if (!half) B(J) = zi[rj];
      }
    });
  }
}

template <typename P, int M, bool kInv, typename OFF, bool kHalfB = false, bool kG = false, typename TW>
__device__ __forceinline__ void pl_set(float* pa, float* pb, bool half, const TW& tw,
                                       typename P::elem* ga = nullptr, typename P::elem* gb = nullptr,
                                       int m0 = 0, uint32_t k65536 = 0) {
  float zr[M], zi[M];
  pl_set_in<P, M, kInv, OFF, kHalfB, kG>(zr, zi, pa, pb, half, tw, ga, gb, m0, k65536);
  pl_set_out<P, M, kInv, OFF, kHalfB, kG>(zr, zi, pa, pb, half, ga, gb, m0);
}

// DC set of pass 3 with a natural-order row on one side (kG): forward H -> row, inverse row -> H;
// the row is the global one (LD = gio1, ST = gio) or the staged one in shared memory (sio1, sst1).
template <typename P, int M, bool kInv, typename OFF, typename LD = gio1<typename P::elem>>
__device__ __forceinline__ void pl_dc_g_in(float (&d)[M], const float* p0, const typename P::elem* g0, int m0,
                                           uint32_t k65536) {
  ct::static_for<0, M>([&](auto J) {
    constexpr int j = decltype(J)::value;
    d[j] = kInv ? LD::ld(g0 + j * m0, k65536) : p0[OFF::a(j)];
  });
  if (!kInv)
    rfft_fwd_reg<M>(d);
  else
    rfft_inv_reg<M>(d);
}
template <typename P, int M, bool kInv, typename OFF, typename ST = gio<typename P::elem>>
__device__ __forceinline__ void pl_dc_g_out(const float (&d)[M], float* p0, typename P::elem* g0, int m0,
                                            float scale) {
  ct::static_for<0, M>([&](auto J) {
    constexpr int j = decltype(J)::value;
    if (!kInv)
      ST::st1(g0 + j * m0, d[j] * scale);
    else
      p0[OFF::a(j)] = d[j] * scale;
  });
}
// pass-2 twiddle: TW2[j][c] (17 columns), indexed by natural j: c = k - 1 (k = 1 .. 15) W_1024^{k rev5(j)};
// c = 15 the paired block-Nyquist sets (k = 16), c = 16 the paired block-DC sets (k = 0, no twiddle).
// Forward: the paired columns carry the factor 1/2 of the two-for-one split (PairFix); inverse: conj.
struct LTw2 {
  static constexpr int kStride = 17;
  const float2* h;  // &TW2[0][c]
  template <int R_>
  __device__ __forceinline__ float2 at() const {
    return h[rev_bits<5>(R_) * kStride];
  }
};

// Pass 2, paired sets (round 2): each 1024-slot window has 15 complex sets (k = 1 .. 15), a real-input
// set of its block Nyquists (k = 16) and a real one of its block DCs (k = 0).  Instead of one lane per
// window running the k = 16 set with a zero imaginary part AND then the DC set as a real FFT (1.5 sets
// of instructions for its whole warp), two windows w1, w2 share one complex 32-point set per kind:
// z = (s1 + i s2) (the twiddle is a scalar, so it applies to the sum), then the two spectra separate by
// symmetry — the DC sets' outputs satisfy X[-q] = conj X[q], the Nyquist sets' U[31 - q] = conj U[q]
// (bins 32 q + 16 of a real 1024-point spectrum).  Every lane then runs exactly one complex set; the
// pair's loads and stores are the regular set code with pa = window w1, pb = window w2 (rebased), and
// only this fix-up differs.  R(q) below = the registers of DFT index q (inverse: at position rev5(q)).
template <int M, bool kInv>
struct PairFix {
  int kind;   // 0: regular set (no-op), 1: paired DC sets, 2: paired Nyquist sets
  float s0;   // forward: scale of the j = 0 input (1/2 for the pairs; the table carries it for j >= 1)
  bool has1;  // inverse: the second set exists (a ragged tile's last pair may have one member only)
  __device__ __forceinline__ void operator()(float (&zr)[M], float (&zi)[M]) const {
    constexpr int LM = ilog2c<M>(), H = M / 2;
    if constexpr (!kInv) {
      const float sc = kind != 0 ? 0.5f : s0;  // (uniform: every lane; regular sets s0 = 1)
      zr[0] *= sc;
      zi[0] *= sc;
    } else if (kind == 1) {
      // loaded: R(q) = (P1[q], P2[M-1-q]) for q < M/2, (P2[M-1-q], -P1[q]) for q >= M/2 (P1 / P2 = the
      // two packed real DC spectra); wanted: R(q) = Z_q = X1_q + i X2_q.
      if (!has1) {
        ct::static_for<0, H>([&](auto Q) {
          constexpr int q = decltype(Q)::value;
          zi[rev_bits<LM>(q)] = 0.f;
          zr[rev_bits<LM>(q + H)] = 0.f;
        });
      }
      float nr[M], ni[M];
      nr[0] = zr[rev_bits<LM>(0)];
      ni[0] = zr[rev_bits<LM>(M - 1)];  // Z_0 = P1[0] + i P2[0]
      nr[H] = -zi[rev_bits<LM>(H)];
      ni[H] = zi[rev_bits<LM>(H - 1)];  // Z_{M/2} = P1[M/2] + i P2[M/2]
      ct::static_for<1, H>([&](auto Q) {
        constexpr int q = decltype(Q)::value, r = M - q;
        const float p1q = zr[rev_bits<LM>(q)], p1r = -zi[rev_bits<LM>(r)];
        const float p2r = zi[rev_bits<LM>(q - 1)], p2q = zr[rev_bits<LM>(M - 1 - q)];
        nr[q] = p1q - p2r;
        ni[q] = p1r + p2q;
        nr[r] = p1q + p2r;
        ni[r] = p2q - p1r;
      });
      ct::static_for<0, M>([&](auto Q) {
        constexpr int q = decltype(Q)::value;
        zr[rev_bits<LM>(q)] = nr[q];
        zi[rev_bits<LM>(q)] = ni[q];
      });
    } else if (kind == 2) {
      // loaded: R(q) = (Re U1_q, Im U2_q), R(M-1-q) = (Re U2_q, -Im U1_q) for q < M/2; wanted Z = U1 + i U2
      ct::static_for<0, H>([&](auto Q) {
        constexpr int q = decltype(Q)::value;
        constexpr int a = rev_bits<LM>(q), b = rev_bits<LM>(M - 1 - q);
        const float u1r = zr[a], u2r = zr[b], mu1i = zi[b];
        const float u2i = has1 ? zi[a] : 0.f;
        const float u2r_ = has1 ? u2r : 0.f;
        zr[a] = u1r - u2i;
        zi[a] = u2r_ - mu1i;
        zr[b] = u1r + u2i;
        zi[b] = u2r_ + mu1i;
      });
    }
  }
};

// Forward pass 2, paired Nyquist sets: Z (natural order, the 1/2 already in) -> in place, the registers
// the regular store code (pl_set_out) writes to the two windows: window 1 slot 32 t + 16 <- (t < 16 ? zr[t]
// : -zi[t]), window 2 slot 32 (31 - t) + 16 <- (t < 16 ? zi[t] : zr[t]).  U1 = Z_q + conj Z_{31-q},
// U2 = -i (Z_q - conj Z_{31-q}); each q < 16 pair maps onto its own four registers.
template <int M>
__device__ __forceinline__ void pair_nyq_fwd_out(float (&zr)[M], float (&zi)[M]) {
  static_assert(M == 32, "pass-2 sets");
  ct::static_for<0, 16>([&](auto Q) {
    constexpr int q = decltype(Q)::value, r = 31 - q;
    const float ar = zr[q], ai = zi[q], br = zr[r], bi = zi[r];
    zr[q] = ar + br;  // Re U1_q
    zi[q] = br - ar;  // Im U2_q
    zi[r] = bi - ai;  // -Im U1_q
    zr[r] = ai + bi;  // Re U2_q
  });
}
// Forward pass 2, paired DC sets, in place for the regular store code with window 2's store base one
// block further (pb = window 2 + 0, so B(M-1-t) = its slot 32 (32 - t)): window 1 slot 32 t <- (t < 16 ?
// zr[t] : -zi[t]), window 2 slot 32 (32 - t) <- (t < 16 ? zi[t] : zr[t]) for t >= 1; window 2's slot 0
// (P2[0], left in zi[0]) is stored by the caller.  X1 = Z_q + conj Z_{-q}, X2 = -i (Z_q - conj Z_{-q}):
// every pair (q, 32 - q) maps onto its own four registers (no permutation: it spilled next to the bf16
// forward's prefetch registers).
template <int M>
__device__ __forceinline__ void pair_dc_fwd_inplace(float (&zr)[M], float (&zi)[M]) {
  static_assert(M == 32, "pass-2 sets");
  {
    const float r0 = zr[0], i0 = zi[0], r16 = zr[16], i16 = zi[16];
    zr[0] = r0 + r0;      // P1[0]
    zi[0] = i0 + i0;      // P2[0] (stored by the caller)
    zr[16] = i16 + i16;   // P2[16]  (window 2 slot 32 * 16 <- zr[16])
    zi[16] = -(r16 + r16);  // -P1[16] (window 1 slot 32 * 16 <- -zi[16])
  }
  ct::static_for<1, 16>([&](auto Q) {
    constexpr int q = decltype(Q)::value, r = 32 - q;
    const float a = zr[q], b = zr[r], c = zi[q], d = zi[r];
    zr[q] = a + b;  // P1[q] = Re X1_q
    zi[r] = d - c;  // -P1[r], P1[r] = Im X1_q = zi_q - zi_r
    zi[q] = b - a;  // P2[r] = Im X2_q  (window 2 slot 32 r <- zi[q])
    zr[r] = c + d;  // P2[q] = Re X2_q  (window 2 slot 32 q <- zr[r])
  });
}
// Cluster-pair cross stage (m = N, the vector has 2N slots), forward: groups k in this CTA's
// quarter, A from window 0 (H0), B from window 1 (H1), outputs straight to the global row xv.
// U groups per batch: all their shared (local and peer) loads first, then the arithmetic and the
// stores — the generic stores would otherwise keep the compiler from hoisting the next group's loads.
template <typename P>
__device__ __forceinline__ void pl_cross_fwd(const float* H0, const float* H1, const float2* TWCa, float2 twb,
                                             typename P::elem* xv, int r, int tid) {
  using T = typename P::elem;
  constexpr int m = P::N, NT = P::NT, Q = m / 4, U = 4;
  static_assert((Q / NT) % U == 0, "cross-stage batches");
#pragma unroll 1
  for (int i0 = 0; i0 < Q / NT; i0 += U) {
    float ar[U], ai[U], br[U], bi[U];
    float2 ta[U];
    ct::static_for<0, U>([&](auto I) {
      constexpr int u = decltype(I)::value;
      const int k = r * Q + tid + NT * (i0 + u);
      const int kk = k == 0 ? m / 2 : k;  // k = 0 is handled below (its mirror slots are not a group)
      ar[u] = H0[P::phys(kk)];
      ai[u] = H0[P::phys(m - kk)];
      br[u] = H1[P::phys(kk)];
      bi[u] = H1[P::phys(m - kk)];
      ta[u] = TWCa[kk >> 7];  // W_{2m}^k = W^{128 a} W^b, b = k % 128 (fixed per thread)
    });
    ct::static_for<0, U>([&](auto I) {
      constexpr int u = decltype(I)::value;
      // no branch in the batch (its reconvergence showed in the stall samples): k = 0 runs the group
      // formula on k = m/2's slots (the loads above) and is overwritten after the loop
      const int k = r * Q + tid + NT * (i0 + u);
      const int kk = k == 0 ? m / 2 : k;
      const float wr = ta[u].x * twb.x - ta[u].y * twb.y, wi = ta[u].x * twb.y + ta[u].y * twb.x;
      const float ur = fmaf(br[u], wr, -bi[u] * wi), ui = fmaf(br[u], wi, bi[u] * wr);
      gio<T>::st1(xv + kk, ar[u] + ur);
      gio<T>::st1(xv + 2 * m - kk, ai[u] + ui);
      gio<T>::st1(xv + m - kk, ar[u] - ur);
      gio<T>::st1(xv + m + kk, ui - ai[u]);
    });
  }
  if (r == 0 && tid == 0) {  // k = 0: (a, b) -> (a + b, a - b); k = m/2: slot m/2 kept, slot 3m/2 negated
    const float a = H0[P::phys(0)], b = H1[P::phys(0)];
    gio<T>::st1(xv, a + b);
    gio<T>::st1(xv + m, a - b);
    gio<T>::st1(xv + m / 2, H0[P::phys(m / 2)]);
    gio<T>::st1(xv + 3 * m / 2, -H1[P::phys(m / 2)]);
  }
}

// Cluster-pair cross stage, inverse (Eq. 7's first stage, with its 1/2): global row -> H0, H1.
// Batched like the forward: U groups' HBM loads in flight before any shared store.
template <typename P>
__device__ __forceinline__ void pl_cross_inv(float* H0, float* H1, const float2* TWCa, float2 twb,
                                             const typename P::elem* xv, int r, int tid, uint32_t k65536) {
  using T = typename P::elem;
  constexpr int m = P::N, NT = P::NT, Q = m / 4, U = 8;
  static_assert((Q / NT) % U == 0, "cross-stage batches");
#pragma unroll 1
  for (int i0 = 0; i0 < Q / NT; i0 += U) {
    float ykr[U], yki[U], ymr[U], ymi[U];
    ct::static_for<0, U>([&](auto I) {
      constexpr int u = decltype(I)::value;
      const int k = r * Q + tid + NT * (i0 + u);
      const int kk = k == 0 ? m / 2 : k;  // k = 0 is handled below (slot 2m - 0 is outside the row)
      ykr[u] = gio1<T>::ld(xv + kk, k65536);
      yki[u] = gio1<T>::ld(xv + 2 * m - kk, k65536);
      ymr[u] = gio1<T>::ld(xv + m - kk, k65536);
      ymi[u] = -gio1<T>::ld(xv + m + kk, k65536);
    });
    ct::static_for<0, U>([&](auto I) {
      constexpr int u = decltype(I)::value;
      // no branch in the batch: k = 0 runs the group formula on k = m/2's slots and is fixed up after
      const int k = r * Q + tid + NT * (i0 + u);
      const int kk = k == 0 ? m / 2 : k;
      const float2 ta = TWCa[kk >> 7];  // conj(W_{2m}^k)
      const float wr = ta.x * twb.x - ta.y * twb.y, wi = ta.x * twb.y + ta.y * twb.x;
      const float dr = 0.5f * (ykr[u] - ymr[u]), di = 0.5f * (yki[u] - ymi[u]);
      H0[P::phys(kk)] = 0.5f * (ykr[u] + ymr[u]);
      H0[P::phys(m - kk)] = 0.5f * (yki[u] + ymi[u]);
      H1[P::phys(kk)] = fmaf(dr, wr, -di * wi);
      H1[P::phys(m - kk)] = fmaf(dr, wi, di * wr);
    });
  }
  if (r == 0 && tid == 0) {  // k = 0 (slots 0, m) and the unpaired slots m/2, 3m/2
    const float s = gio1<T>::ld(xv, k65536), d = gio1<T>::ld(xv + m, k65536);
    H0[P::phys(0)] = 0.5f * (s + d);
    H1[P::phys(0)] = 0.5f * (s - d);
    H0[P::phys(m / 2)] = gio1<T>::ld(xv + m / 2, k65536);
    H1[P::phys(m / 2)] = -gio1<T>::ld(xv + 3 * m / 2, k65536);
  }
}

// Cluster pair, pass 1: elements 4 g + r and 4 g + 2 + r of the row (the two subsequences 2c, 2c + 1 of
// this CTA's half x[r :: 2]) from one 8-byte (bf16) / 16-byte (fp32) load of the 4-element group at p —
// half the load instructions of two strided scalar loads; the peer CTA uses the other two elements.
template <typename T>
struct pair_ld;
template <>
struct pair_ld<__nv_bfloat16> {
  __device__ __forceinline__ static float2 ld(const __nv_bfloat16* p, uint32_t sel) {
    const uint2 u = __ldcs(reinterpret_cast<const uint2*>(p));
    return make_float2(__uint_as_float(__byte_perm(u.x, 0u, sel)), __uint_as_float(__byte_perm(u.y, 0u, sel)));
  }
  // selector: result bytes (0, 0, e_r lo, e_r hi), e_r = bytes 2r, 2r + 1 of the word
  __device__ __forceinline__ static uint32_t sel(int r) { return r ? 0x3244u : 0x1044u; }
};
template <>
struct pair_ld<float> {
  __device__ __forceinline__ static float2 ld(const float* p, uint32_t sel) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(p));
    return sel ? make_float2(v.y, v.w) : make_float2(v.x, v.z);
  }
  __device__ __forceinline__ static uint32_t sel(int r) { return (uint32_t)r; }
};

// Pass 3's block-DC set (a real M3-point DFT, M3 <= 32) as a warp-cooperative radix-2 DIT over lanes
// (round 2): lane l holds element l in bit-reversed input order, stage h exchanges with lane l ^ h by
// shuffles and applies W_{2h}^{l mod h} = W_32^{(l mod h) 32 / 2h} from a 16-entry table; lane q ends with
// X_q (natural order; inverse: conjugate twiddles, unscaled).  It replaces the real FFT that the thread of
// the zero-imaginary set ran after that set, which made its warp — at n = 32768, with one set per thread,
// the whole CTA at the barrier after pass 3 — wait 1.5 sets' time.
template <int M, bool kInv>
__device__ __forceinline__ float2 dc_warp_dit(float2 v, int lane, const float2* W32) {
#pragma unroll
  for (int h = 1; h < M; h <<= 1) {
    const float pr = __shfl_xor_sync(0xffffffffu, v.x, h);
    const float pi = __shfl_xor_sync(0xffffffffu, v.y, h);
    const bool up = (lane & h) != 0;
    const float ar = up ? pr : v.x, ai = up ? pi : v.y;  // lower element of the pair
    const float br = up ? v.x : pr, bi = up ? v.y : pi;  // upper element
    float2 w = W32[(lane & (h - 1)) * (16 / h)];
    if (kInv) w.y = -w.y;
    const float tr = fmaf(br, w.x, -bi * w.y), ti = fmaf(br, w.y, bi * w.x);
    v = up ? make_float2(ar - tr, ai - ti) : make_float2(ar + tr, ai + ti);
  }
  return v;
}

// Split cluster barrier (the pair's write-after-read hand-off): arrive after this CTA's last read of the
// peer's / its own H, wait just before the next write into H, so the barrier latency overlaps the work in
// between (the next pass 1's loads and register FFT; the inverse pass 1's FFT and stores) instead of a
// full cluster.sync() at the end of every vector.
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// NC = 1: one vector of n = N per CTA.  NC = 2: one vector of n = 2N per cluster pair (see header).
template <typename P, bool kInv, int NC = 1>
__global__ void __launch_bounds__(P::NT, P::MINB) rdfftl_kernel(typename P::elem* __restrict__ x, int64_t batch) {
  using T = typename P::elem;
  constexpr int N = P::N, NT = P::NT, R = P::R, S = P::S, K3 = P::K3, M3 = P::M3;
  static_assert(NC == 1 || NC == 2, "cluster size");
  extern __shared__ float4 smem4[];
  unsigned char* base = reinterpret_cast<unsigned char*>(smem4);
  float* H = reinterpret_cast<float*>(base);
  float2* TW2 = reinterpret_cast<float2*>(base + P::TW2_OFF);
  float2* TW3 = reinterpret_cast<float2*>(base + P::TW3_OFF);
  const int tid = threadIdx.x;
  const float sg = kInv ? 1.0f : -1.0f;
  // cluster pair: rank r holds window r (the n/2-point spectrum of x[r :: 2]); the peer's H via DSMEM
  const int r = NC == 2 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  float* Hpeer = H;
  float2* TWCa = reinterpret_cast<float2*>(base + P::TWC_OFF);
  float2 twb = make_float2(1.f, 0.f);
  if constexpr (NC == 2) {
    Hpeer = cooperative_groups::this_cluster().map_shared_rank(H, r ^ 1);
    for (int e = tid; e < P::TWCA; e += NT) {
      float s, c;
      sincospif(2.0f * (float)(128 * e) / (float)(2 * N), &s, &c);
      TWCa[e] = make_float2(c, sg * s);
    }
    float s, c;
    sincospif(2.0f * (float)(tid % 128) / (float)(2 * N), &s, &c);
    twb = make_float2(c, sg * s);
  }
  float* H0 = r == 0 ? H : Hpeer;
  float* H1 = r == 0 ? Hpeer : H;
  constexpr int64_t NV = (int64_t)N * NC;  // elements per vector
  constexpr int XS = NC;                   // element stride of this CTA's half in the row
  // pass 2 runs paired DC / Nyquist sets (PairFix, pair_dc_fwd_inplace / pair_nyq_fwd_out) in every
  // (n, direction, dtype) cell: faster or equal everywhere once pass 3's DC set moved to a warp of its own
  // (the bf16 n = 32768 inverse 0.320 -> 0.333 of HBM, r02_v41; before that it had measured slower, r02_v31)
  for (int e = tid; e < 32 * LTw2::kStride; e += NT) {  // LTw2's 17 columns (paired ones: 1/2 in the forward)
    const int j = e / LTw2::kStride, col = e % LTw2::kStride;
    const int k = col == 16 ? 0 : col + 1;
    const float h = (!kInv && col >= 15) ? 0.5f : 1.0f;
    float s, c;
    sincospif(2.0f * (float)(k * rev_bits<5>(j)) / 1024.0f, &s, &c);
    TW2[e] = make_float2(h * c, h * sg * s);
  }
  const float2* W32 = TW2 + 32 * LTw2::kStride;  // W_32^t, t < 16 (forward sign; dc_warp_dit conjugates)
  for (int t = tid; t < 16; t += NT) {
    float s, c;
    sincospif((float)t / 16.0f, &s, &c);
    TW2[32 * LTw2::kStride + t] = make_float2(c, -s);
  }
  for (int e = tid; e < P::TW3N; e += NT) {
    const int a = e / K3, k = 1 + e % K3;
    float s, c;
    sincospif(2.0f * (float)(4 * k * a) / (float)N, &s, &c);
    TW3[e] = kInv ? make_float2(c * (1.0f / N), s * (1.0f / N)) : make_float2(c, -s);
  }
  // pass-3 sets k3 = tid + NT i (i < K3PT); k3 = 0 stands for the zero-imaginary set k3 = 512
  // plus the DC set (two real-input sets ~ one complex set of work)
  auto tw3_for = [&](int k3) {  // W^{k}: one sincospif; W^{2k}, W^{3k} by products (~2-3 ulp)
    LTw3<K3> t;
    t.h = TW3 + (k3 - 1);
    float s, c;
    sincospif(2.0f * (float)k3 / (float)N, &s, &c);
    const float2 w = make_float2(c, sg * s);
    t.w1 = w;
    t.w2 = make_float2(fmaf(w.x, w.x, -w.y * w.y), 2.0f * w.x * w.y);
    t.w3 = make_float2(fmaf(t.w2.x, w.x, -t.w2.y * w.y), fmaf(t.w2.x, w.y, t.w2.y * w.x));
    return t;
  };
  // pass 3; one-CTA plan (NC = 1): the forward stores its outputs straight to the row xv and the
  // inverse reads its inputs straight from it (no chunked H <-> HBM phase: two passes of shared
  // traffic fewer per vector); the cluster pair keeps them in H for the cross stage.
  constexpr bool kG3 = (NC == 1);
  // the staged forward costs 2 more barriers per vector: slower at one CTA per SM (n = 32768)
  constexpr bool kST = (NC == 1 && P::kST && (kInv || P::MINB > 1));
  const uint32_t k65536 = kTwo16;
  T* SR = reinterpret_cast<T*>(H);  // kST: the staged natural-order row (aliases H)
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + P::BAR_OFF);
  // pass 3's DC set: the last warp, cooperatively (dc_warp_dit).  Its natural-order side is the global row
  // (one-CTA plan), the staged row SR (kST) or H (cluster pair); its H side is slots OffP3::a(j).
  // (kDCW off: the bf16 n = 8192 forward, whose staged pass 3 spills with the warp's two extra registers
  // next to its prefetch and pass-2 pairs; there the zero-imaginary set's thread runs the DC set too)
  constexpr bool kDCW = !(N == 8192 && sizeof(T) == 2 && !kInv && kST);
  constexpr int LM3 = ilog2c<M3>();
  const bool dcw = kDCW && tid >= NT - 32;
  const int dl = tid & 31;
  auto dc_row_ld = [&](const T* row, int s_) -> float {
    if constexpr (NC == 2) return H[OffP3<P>::a(s_)];
    else if constexpr (kST) return sio1<T>::ld(SR + 1024 * s_, k65536);
    else return gio1<T>::ld(row + 1024 * s_, k65536);
  };
  auto dc_row_st = [&](T* row, int s_, float val) {
    if constexpr (NC == 2) H[OffP3<P>::a(s_)] = val;
    else if constexpr (kST) sst1<T>::st1(SR + 1024 * s_, val);
    else gio<T>::st1(row + 1024 * s_, val);
  };
  auto dc_in = [&](auto inv, const T* row) -> float2 {  // (the whole DC warp)
    constexpr bool kI = decltype(inv)::value;
    float2 v = make_float2(0.f, 0.f);
    if (dl < M3) {
      if constexpr (!kI) {
        v.x = H[OffP3<P>::a(dl)];  // element dl in bit-reversed order (the per-stage invariant)
      } else {  // X_q, q = rev(dl), from the packed spectrum (X_{M-q} = conj X_q)
        const int q = (int)(__brev((unsigned)dl) >> (32 - LM3));
        const int qa = q <= M3 / 2 ? q : M3 - q;
        const float re = dc_row_ld(row, qa);
        const float im = (qa == 0 || qa == M3 / 2) ? 0.f : dc_row_ld(row, M3 - qa);
        v = make_float2(re, q <= M3 / 2 ? im : -im);
      }
    }
    return dc_warp_dit<M3, kI>(v, dl, W32);
  };
  auto dc_out = [&](auto inv, T* row, float2 v) {
    constexpr bool kI = decltype(inv)::value;
    if (dl < M3) {
      if constexpr (!kI) {  // packed: slot 1024 q <- Re X_q (q <= M/2), slot 1024 (M - q) <- Im X_q
        if (dl <= M3 / 2) dc_row_st(row, dl, v.x);
        if (dl >= 1 && dl < M3 / 2) dc_row_st(row, M3 - dl, v.y);
      } else {  // x_t (times M, unscaled) -> H slot rev(t), scaled by 1/N
        H[OffP3<P>::a((int)(__brev((unsigned)dl) >> (32 - LM3)))] = v.x * (1.0f / N);
      }
    }
  };
  auto pass3 = [&](auto inv, T* xv) {
    constexpr bool kI = decltype(inv)::value;
    if constexpr (kST) {
      // sets k = tid + NT i, i < K3PT (tid 0, i = 0: the zero-imaginary set k = 512 and the DC set); the
      // staged row SR in place of the global one.  zr/zi carry the results across the barrier; tid 0
      // packs its DC set into the registers its half set leaves free (forward: zr/zi[M3/2 ..]; inverse:
      // zi) so the live set across the barrier stays 2 K3PT M3 floats on every path.
      using SIO = sio1<T>;
      using SST = sst1<T>;
      constexpr int KP = P::K3PT;
      float zr[KP][M3], zi[KP][M3];
      ct::static_for<0, KP>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int kk = tid + NT * i;
        if (i == 0 && kk == 0) {  // the zero-imaginary set (the DC set: the last warp, below)
          pl_set_in<P, M3, kI, OffP3<P>, true, true, SIO>(zr[i], zi[i], H + K3, H - K3, true, tw3_for(K3), SR + K3,
                                                          SR - K3, 1024, k65536);
          if constexpr (!kDCW) {  // ... or this thread: its DC results in the registers the half set leaves free
            float d[M3];
            pl_dc_g_in<P, M3, kI, OffP3<P>, SIO>(d, H, SR, 1024, k65536);
            ct::static_for<0, M3>([&](auto J) {
              constexpr int j = decltype(J)::value;
              if constexpr (kI) zi[i][j] = d[j];
              else if constexpr (j < M3 / 2) zr[i][M3 / 2 + j] = d[j];
              else zi[i][j] = d[j];
            });
          }
        } else {
          pl_set_in<P, M3, kI, OffP3<P>, false, true, SIO>(zr[i], zi[i], H + kk, H - kk, false, tw3_for(kk),
                                                           SR + kk, SR - kk, 1024, k65536);
        }
      });
      float2 dcv = make_float2(0.f, 0.f);
      if (dcw) dcv = dc_in(inv, xv);
      __syncthreads();  // every set read: H / SR free for the writes
      if (dcw) dc_out(inv, xv, dcv);
      ct::static_for<0, KP>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int kk = tid + NT * i;
        if (i == 0 && kk == 0) {
          if constexpr (!kDCW) {
            float d[M3];
            ct::static_for<0, M3>([&](auto J) {
              constexpr int j = decltype(J)::value;
              if constexpr (kI) d[j] = zi[i][j];
              else if constexpr (j < M3 / 2) d[j] = zr[i][M3 / 2 + j];
              else d[j] = zi[i][j];
            });
            pl_set_out<P, M3, kI, OffP3<P>, true, true, SST>(zr[i], zi[i], H + K3, H - K3, true, SR + K3, SR - K3,
                                                             1024);
            pl_dc_g_out<P, M3, kI, OffP3<P>, SST>(d, H, SR, 1024, kI ? 1.0f / N : 1.0f);
          } else {
            pl_set_out<P, M3, kI, OffP3<P>, true, true, SST>(zr[i], zi[i], H + K3, H - K3, true, SR + K3, SR - K3,
                                                             1024);
          }
        } else {
          pl_set_out<P, M3, kI, OffP3<P>, false, true, SST>(zr[i], zi[i], H + kk, H - kk, false, SR + kk, SR - kk,
                                                            1024);
        }
      });
      return;
    }
#pragma unroll 1
    for (int i = 0; i < P::K3PT; ++i) {
      const int kk = tid + NT * i;
      if (kk == 0) {  // the zero-imaginary set k = 512 (the DC set: the last warp, below)
        pl_set<P, M3, kI, OffP3<P>, true, kG3>(H + K3, H - K3, true, tw3_for(K3), xv + K3, xv - K3, 1024, k65536);
      } else {
        pl_set<P, M3, kI, OffP3<P>, false, kG3>(H + kk, H - kk, false, tw3_for(kk), xv + kk, xv - kk, 1024,
                                                k65536);
      }
    }
    if (dcw) dc_out(inv, xv, dc_in(inv, xv));  // (every lane loads before any lane stores: in place is safe)
  };
  // pass-2 lane: window ww, k2 = 1 .. 15; lane 0 of each half-warp: a paired DC or Nyquist set (below)
  // The two half-warps take blocks ww and ww + D, D = n/4096: their pads then differ by 16 floats
  // (4 pad periods), so the half-warps' scalar accesses fall on complementary bank halves (with
  // adjacent blocks they overlapped: 2-way conflicts on every pass-2 access).
  constexpr int D2 = N / 4096;
  const int w32 = tid / 32, hw = (tid / 16) & 1;
  const int ww = (w32 % D2) + (w32 / D2) * 2 * D2 + hw * D2, k2 = tid % 16;
  const bool act2 = tid < P::NW2 * 16;
  float* h2 = H + P::phys(ww * 1024);  // block base (pad of the block start; OffP2 adds the rest)
  // lanes k2 = 1 .. 15: set k2 of window ww; lane k2 = 0 of each half-warp: a paired set (PairFix) of the
  // warp's two windows w1 = ww(hw 0), w2 = w1 + D2 — block DCs on half-warp 0, block Nyquists on half-warp
  // 1.  Their slots 32 j (+ 16) then fall on the two banks the 30 regular lanes leave free (the half-warps'
  // pads differ by 16 floats): a pairing across other windows put a 2-way conflict on every pass-2 access.
  const int pkind = k2 != 0 ? 0 : (hw == 0 ? 1 : 2);
  float* pa2 = h2 + k2;
  float* pb2 = h2 - k2;
  LTw2 tw2;
  tw2.h = TW2 + (k2 - 1);
  if (pkind != 0) {
    float* hw1 = H + P::phys((ww - hw * D2) * 1024);
    float* hw2 = H + P::phys((ww - hw * D2 + D2) * 1024);
    pa2 = pkind == 1 ? hw1 : hw1 + 16;       // A(j): window 1 slot 32 j (+ 16)
    pb2 = pkind == 1 ? hw2 - 32 : hw2 - 16;  // B(j) = pb[32 (j + 1)]: window 2 slot 32 j (+ 16)
    tw2.h = TW2 + (pkind == 1 ? 16 : 15);
  }
  const PairFix<32, kInv> pfix{pkind, 1.0f, true};
  if (kST && tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  // kST inverse: the row of vector vv -> SR (TMA bulk load; 4 copies of N/4 elements)
  auto issue_row = [&](int64_t vv) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, (uint32_t)(N * sizeof(T)));
    ct::static_for<0, 4>([&](auto C) {
      constexpr int c = decltype(C)::value;
      bulk_g2s(SR + c * (N / 4), x + vv * NV + c * (N / 4), (uint32_t)(N / 4 * sizeof(T)), bar);
    });
  };
  __syncthreads();
  if constexpr (NC == 2) cooperative_groups::this_cluster().sync();  // peer's H mapped and live
  if constexpr (kST && kInv) {
    if (tid == 0 && (int64_t)blockIdx.x < batch) issue_row(blockIdx.x);
  }
  uint32_t it = 0;
  // bf16 forward, one vector per CTA: pass 1's element pairs of the NEXT vector are loaded into
  // registers (32 raw bf16x2 words per thread) right after this vector's pass 1, so their HBM latency
  // hides behind passes 2 and 3 instead of stalling the next pass 1
  constexpr bool kPF = (NC == 1 && sizeof(T) == 2 && !kInv);
  uint32_t pf[kPF ? R : 1];
  if constexpr (kPF) {
    if (tid < S / 2 && (int64_t)blockIdx.x < batch) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(x + (int64_t)blockIdx.x * NV) + tid;
      ct::static_for<0, R>([&](auto I) { pf[decltype(I)::value] = __ldcs(src + (S / 2) * decltype(I)::value); });
    }
  }
  const uint32_t psel = pair_ld<T>::sel(r);
  for (int64_t v = blockIdx.x / NC; v < batch; v += gridDim.x / NC, ++it) {
    T* xv = x + v * NV;
    T* xh = xv + r;  // this CTA's half: elements xh[XS * e], e < N
    if (!kInv) {
      if (tid < S / 2) {  // pass 1: subsequences 2c, 2c+1 -> windows rev(2c), rev(2c) + S/2
        const int c = tid;
        float2 b[R];
        ct::static_for<0, R>([&](auto I) {
          constexpr int i = decltype(I)::value;
          if constexpr (kPF)
            b[rev_bits<5>(i)] = make_float2(__uint_as_float(pf[i] * k65536), __uint_as_float(pf[i] & 0xffff0000u));
          else if constexpr (NC == 1)
            b[rev_bits<5>(i)] = gio<T>::ld2(xv + 2 * c + S * i, k65536);
          else  // x[r :: 2] at 2 (2c + S i) and 2 (2c + 1 + S i): the group of 4 at 4c + 2 S i
            b[rev_bits<5>(i)] = pair_ld<T>::ld(xv + 4 * c + 2 * S * i, psel);
        });
        if constexpr (kPF) {
          const int64_t vn = v + gridDim.x;
          if (vn < batch) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(x + vn * NV) + c;
            ct::static_for<0, R>([&](auto I) { pf[decltype(I)::value] = __ldcs(src + (S / 2) * decltype(I)::value); });
          }
        }
        rfft_fwd_reg<R>(b);
        if constexpr (NC == 2) {  // the peer has finished the previous vector's cross stage (reads of this H)
          if (it > 0) cluster_wait_acquire();
        }
        if constexpr (kST) {  // the previous vector's bulk store still reads SR (= H)
          if (tid == 0) bulk_wait_read<0>();
          __syncthreads();  // (kST: S / 2 == NT, every thread is here)
        }
        const int w0 = rev_bits<P::LS>(2 * c), w1 = w0 + S / 2;
        float* h0 = H + P::phys(w0 * 32);  // a window never crosses a pad boundary
        float* h1 = H + P::phys(w1 * 32);
        ct::static_for<0, R / 4>([&](auto I) {
          constexpr int i = 4 * decltype(I)::value;
          *reinterpret_cast<float4*>(h0 + i) = make_float4(b[i].x, b[i + 1].x, b[i + 2].x, b[i + 3].x);
          *reinterpret_cast<float4*>(h1 + i) = make_float4(b[i].y, b[i + 1].y, b[i + 2].y, b[i + 3].y);
        });
      }
      __syncthreads();
      {
        if (act2) {
          float zr[32], zi[32];
          pl_set_in<P, 32, false, OffP2<P>>(zr, zi, pa2, pb2, false, tw2, nullptr, nullptr, 0, 0u, pfix);
          if (pkind == 1) pair_dc_fwd_inplace(zr, zi);
          else if (pkind == 2) pair_nyq_fwd_out(zr, zi);
          // one store sequence for every lane (the DC pair's window-2 base one block further)
          pl_set_out<P, 32, false, OffP2<P>>(zr, zi, pa2, pb2 + (pkind == 1 ? 32 : 0), false, nullptr, nullptr, 0,
                                             pkind == 1);
          if (pkind == 1) {  // window 2 slots 0 and 32 * 16: P2[0], P2[16]
            (pb2 + 32)[OffP2<P>::a(0)] = zi[0];
            (pb2 + 32)[OffP2<P>::a(16)] = zr[16];
          }
        }
      }
      __syncthreads();
      pass3(std::false_type{}, xv);
      if constexpr (kST) {
        fence_proxy_async_smem();  // SR's generic writes before the bulk store reads them
        __syncthreads();
        if (tid == 0) {
          ct::static_for<0, 4>([&](auto C) {
            constexpr int c = decltype(C)::value;
            bulk_s2g(xv + c * (N / 4), SR + c * (N / 4), (uint32_t)(N / 4 * sizeof(T)));
          });
          bulk_commit();
        }
      } else if constexpr (NC == 1) {
        __syncthreads();  // H is read by pass 3 until here; the next vector's pass 1 writes it
      } else {
        cooperative_groups::this_cluster().sync();  // both windows complete and visible
        pl_cross_fwd<P>(H0, H1, TWCa, twb, xv, r, tid);
        cluster_arrive_release();  // this CTA is done reading both H; the wait sits before the next H write
      }
    } else {
      if constexpr (NC == 2) {
        if (it > 0) cluster_wait_acquire();  // the peer has read its H (the previous vector's pass 1)
        pl_cross_inv<P>(H0, H1, TWCa, twb, xv, r, tid, k65536);
        cooperative_groups::this_cluster().sync();  // both windows written (half of each remotely)
      }
      if constexpr (kST) mbar_wait(bar, it & 1);  // this vector's row staged in SR
      pass3(std::true_type{}, xv);  // NC = 1: reads the row straight from HBM (kST: from SR)
      __syncthreads();
      if (act2) {
        float zr[32], zi[32];
        pl_set_in<P, 32, true, OffP2<P>>(zr, zi, pa2, pb2, false, tw2, nullptr, nullptr, 0, 0u, pfix);
        pl_set_out<P, 32, true, OffP2<P>>(zr, zi, pa2, pb2, false);
      }
      __syncthreads();
      if (tid < S / 2) {  // inverse pass 1
        const int c = tid;
        const int w0 = rev_bits<P::LS>(2 * c), w1 = w0 + S / 2;
        const float* h0 = H + P::phys(w0 * 32);
        const float* h1 = H + P::phys(w1 * 32);
        float2 b[R];
        ct::static_for<0, R / 4>([&](auto I) {
          constexpr int i = 4 * decltype(I)::value;
          const float4 f0 = *reinterpret_cast<const float4*>(h0 + i);
          const float4 f1 = *reinterpret_cast<const float4*>(h1 + i);
          b[i] = make_float2(f0.x, f1.x);
          b[i + 1] = make_float2(f0.y, f1.y);
          b[i + 2] = make_float2(f0.z, f1.z);
          b[i + 3] = make_float2(f0.w, f1.w);
        });
        if constexpr (kST) {  // H read: the next vector's row may land in SR (= H)
          __syncthreads();
          if (tid == 0 && v + gridDim.x < batch) issue_row(v + gridDim.x);
        }
        if constexpr (NC == 2) cluster_arrive_release();  // H read; the wait sits before the next cross stage
        rfft_inv_reg<R>(b);
        ct::static_for<0, R>([&](auto I) {
          constexpr int i = decltype(I)::value;
          if constexpr (NC == 1) {
            gio<T>::st2(xv + 2 * c + S * i, b[rev_bits<5>(i)]);
          } else {
            gio<T>::st1(xh + XS * (2 * c + S * i), b[rev_bits<5>(i)].x);
            gio<T>::st1(xh + XS * (2 * c + 1 + S * i), b[rev_bits<5>(i)].y);
          }
        });
      }
      if constexpr (kST) {
        // no barrier: H was released after pass 1's reads, and the next vector's pass 3 writes H only
        // after its own barrier
      } else if constexpr (NC == 1) {
        __syncthreads();
      }
    }
  }
  if constexpr (NC == 2) {  // match the last arrive: the peer may still read this CTA's H
    if (it > 0) cluster_wait_acquire();
  }
  if constexpr (kST && !kInv) {
    if (tid == 0) bulk_wait<0>();
  }
}

template <typename P>
bool launch_planl(typename P::elem* x, int64_t batch, bool inverse, int sms, cudaStream_t st) {
  auto kf = rdfftl_kernel<P, false>;
  auto ki = rdfftl_kernel<P, true>;
  static int per_sm_dev[kMaxDevices] = {};
  int& per_sm = per_sm_dev[device_index()];
  if (!per_sm) {
    for (auto k : {kf, ki}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::BYTES);
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    }
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, kf, P::NT, P::BYTES);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ki, P::NT, P::BYTES);
    per_sm = a < b ? a : b;
    if (per_sm < 1) per_sm = 1;
    if (verbose())
      std::fprintf(stderr, "[rdfft] planL n=%d: %zu B smem, %d threads, %d CTAs/SM\n", P::N, (size_t)P::BYTES, P::NT,
                   per_sm);
  }
  const int grid = (int)(batch < (int64_t)per_sm * sms ? batch : (int64_t)per_sm * sms);
  if (inverse)
    ki<<<grid, P::NT, P::BYTES, st>>>(x, batch);
  else
    kf<<<grid, P::NT, P::BYTES, st>>>(x, batch);
  return true;
}

// n = 2 N on cluster pairs (P = PlanL<T, N>, N = 32768 -> n = 65536): one pair per 2 SMs.
template <typename P>
bool launch_planl_pair(typename P::elem* x, int64_t batch, bool inverse, int sms, cudaStream_t st) {
  auto kf = rdfftl_kernel<P, false, 2>;
  auto ki = rdfftl_kernel<P, true, 2>;
  static bool configured_dev[kMaxDevices] = {};
  bool& configured = configured_dev[device_index()];
  if (!configured) {
    for (auto k : {kf, ki}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::BYTES2);
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    }
    configured = true;
    if (verbose())
      std::fprintf(stderr, "[rdfft] planL pair n=%d: %zu B smem per CTA, %d threads, cluster 2\n", 2 * P::N,
                   (size_t)P::BYTES2, P::NT);
  }
  const int64_t pairs = batch < (int64_t)(sms / 2) ? batch : (int64_t)(sms / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(P::NT);
  cfg.dynamicSmemBytes = P::BYTES2;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = inverse ? cudaLaunchKernelEx(&cfg, ki, x, batch) : cudaLaunchKernelEx(&cfg, kf, x, batch);
  return e == cudaSuccess;
}

}  // namespace rdfft
