/*
 * rdfft.h — C-ABI of librdfft.so: the B200 (sm_100a) hot path of rdFFT,
 * "in-place real-domain FFT" (arXiv 2511.01385).
 *
 * Citations: P:Lxxx = PAPER.md line; readings C1..C16 are listed in DESIGN.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Pointers x, a, b, w, y, g, dx, dw are DEVICE pointers (cudaMalloc / torch
 *    CUDA tensors).  Buffers are row-major with contiguous rows: a batch of
 *    vectors is [batch][n]; BCA activations are [T][d] with each row made of
 *    d/p consecutive length-p blocks (reading C14).
 *  - dtype is RDFFT_F32 (IEEE fp32) or RDFFT_BF16 (bfloat16 storage).  All
 *    arithmetic is fp32 in registers; bf16 results are rounded to nearest even
 *    on store (reading C7).  dw is always fp32.
 *  - n (the transform length) is a power of two with 2 <= n <= 65536; the BCA
 *    block size p is a power of two with 2 <= p <= 4096 (reading C9; the paper
 *    runs p = 128 .. 4096; n = 8192 .. 65536 is SURVEY
 *    §8(f) N2: one vector per CTA in shared memory up to 32768, n = 65536 on a
 *    thread-block cluster of two CTAs exchanging the last stage through
 *    distributed shared memory).
 *  - stream is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous on that stream; inputs are validated synchronously on the
 *    host before anything is launched, and nothing is launched on error.
 *  - Ownership: the caller owns every buffer.  The library allocates NO device
 *    or host memory per call (no scratch, no plan object, no hidden state);
 *    twiddle factors are generated on chip.  One buffer must not be used by
 *    two concurrent calls.
 *  - Base pointers must be 16-byte aligned (torch allocations are 256 B); the
 *    kernels use 128-bit accesses.  Any batch, including ragged tails, is
 *    handled.
 *  - batch == 0 (or T == 0) is a successful no-op.
 *  - Non-finite inputs are not checked; IEEE propagation applies.
 *  - Return value: rdfft_status_t.  RDFFT_E_CUDA reports a launch error
 *    (cudaGetLastError after launch); asynchronous faults surface on the
 *    stream as usual.
 *
 * Packed layout ("Squeeze N+2 into N" / "Memory Layout Design"):
 *    slot 0 = Re y_0,  slot n/2 = Re y_{n/2},
 *    slot k = Re y_k,  slot n-k = Im y_k   for 1 <= k < n/2   (reading C2),
 *  with y_k = sum_t x_t exp(-2 pi i k t / n)  (Eq. 1; reading C3).
 */
#ifndef RDFFT_H
#define RDFFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { RDFFT_F32 = 0, RDFFT_BF16 = 1 } rdfft_dtype_t;

typedef enum {
  RDFFT_OK = 0,
  RDFFT_E_SIZE = 1,  /* n not a power of two in [2, 65536] (p: [2, 4096])        */
  RDFFT_E_NULL = 2,  /* null pointer with a non-empty batch                       */
  RDFFT_E_ALIGN = 3, /* a base pointer is not 16-byte aligned                     */
  RDFFT_E_DTYPE = 4, /* dtype not RDFFT_F32 / RDFFT_BF16                          */
  RDFFT_E_SHAPE = 5, /* negative batch, b_batch not in {1, batch}, d % p != 0     */
  RDFFT_E_ALIAS = 6, /* forbidden overlap between buffers (see each call)         */
  RDFFT_E_CUDA = 7   /* the kernel launch failed                                  */
} rdfft_status_t;

/* rdfft_fwd — batched in-place forward rdFFT (§4.1, Prop. 1).
 *   x: [batch][n] real signals of `dtype`, overwritten by their packed spectra.
 *   Equals pack(DFT(x)) row by row; touches no memory outside x.            */
int rdfft_fwd(void* x, int64_t batch, int64_t n, int dtype, void* stream);

/* rdfft_inv — batched in-place inverse rdFFT (§4.2, Eq. 7).
 *   x: [batch][n] packed spectra, overwritten by the real signals
 *   x_t = (1/n) sum_k y_k exp(+2 pi i k t / n)  (1/n included, reading C4). */
int rdfft_inv(void* x, int64_t batch, int64_t n, int dtype, void* stream);

/* rdfft_packed_mul — a <- a (.) b per frequency bin, in the packed domain
 * (the product of Hermitian spectra stays Hermitian).
 *   a: [batch][n] packed spectra (in/out); b: [b_batch][n] packed spectra,
 *   read only, b_batch == 1 broadcasts b to every row of a.
 *   b may not overlap a unless b == a and b_batch == batch (RDFFT_E_ALIAS).  */
int rdfft_packed_mul(void* a, const void* b, int64_t batch, int64_t n, int64_t b_batch, int dtype,
                     void* stream);

/* rdfft_packed_conjmul — a <- a (.) conj(b) per bin (Eq. 5 products).
 *   Same arguments and rules as rdfft_packed_mul.                            */
int rdfft_packed_conjmul(void* a, const void* b, int64_t batch, int64_t n, int64_t b_batch, int dtype,
                         void* stream);

/* bca_fwd — fused block-circulant adapter forward (Eq. 4).
 *   x: [T][d_in] (read only, NOT modified: reading C13)
 *   w: [q_out][q_in][p] time-domain first columns c_ij (reading C10, C12),
 *      q_in = d_in/p, q_out = d_out/p, same dtype as x
 *   y: [T][d_out] output, y_i = sum_j circ(w_ij) x_j = IrdFFT(sum_j W_ij (.) X_j)
 *   y may not overlap x or w (RDFFT_E_ALIAS).  d_in % p, d_out % p must be 0. */
int bca_fwd(const void* x, const void* w, void* y, int64_t T, int64_t d_in, int64_t d_out, int64_t p,
            int dtype, void* stream);

/* bca_fwd_accum — bca_fwd that ADDS the adapter output to y's contents:
 *   y <- y + IrdFFT(sum_j W_ij (.) X_j)
 * i.e. the frozen path's output W0 x (already in y) plus the block-circulant
 * adapter in the same pass, as the adapter is used in fine-tuning
 * (SURVEY §8(f) N4 "y += fusion").  y is read and written
 * once per element (fp32 add, then the usual RNE store for bf16).  Same
 * arguments and aliasing rules as bca_fwd.                                  */
int bca_fwd_accum(const void* x, const void* w, void* y, int64_t T, int64_t d_in, int64_t d_out, int64_t p,
                  int dtype, void* stream);

/* bca_bwd — fused block-circulant adapter backward (Eq. 5, P:L174-183;
 * blockwise pairing reading C11).  With G_i = rdFFT(g_i), X_j = rdFFT(x_j),
 * W_ij = rdFFT(w_ij):
 *   dx_j  = IrdFFT( sum_i conj(W_ij) (.) G_i )              -> dx [T][d_in]
 *   dw_ij = IrdFFT( sum_t conj(X_tj) (.) G_ti )             -> dw [q_out][q_in][p] fp32
 *   x, w, g: as in bca_fwd (g = dL/dy, [T][d_out]).
 *   dx may alias g exactly when d_in == d_out ("overwriting the grad_output
 *   in-place"); any other overlap of dx with x, w, g is RDFFT_E_ALIAS.
 *   dw (fp32, 16-byte aligned) is OVERWRITTEN (zeroed on the stream, then
 *   accumulated); it must not overlap anything.  Accumulation over tokens uses
 *   fp32 atomics, so dw is reproducible only to rounding, not bitwise.      */
int bca_bwd(const void* x, const void* w, const void* g, void* dx, float* dw, int64_t T, int64_t d_in,
            int64_t d_out, int64_t p, int dtype, void* stream);

/* bca_bwd_accum — bca_bwd that ADDS this call's weight gradient to dw instead of
 * overwriting it (gradient accumulation over micro-batches; the paper trains
 * with accumulation 4).  Same arguments, aliasing rules and dx as
 * bca_bwd.  dw's old contents are first forward-transformed in place (fp32
 * rdFFT, exact up to one round trip, ~1e-7 relative), the new spectra are
 * accumulated on top and the usual in-place inverse finishes:
 *   dw <- dw + IrdFFT( sum_t conj(X_tj) (.) G_ti ).                          */
int bca_bwd_accum(const void* x, const void* w, const void* g, void* dx, float* dw, int64_t T, int64_t d_in,
                  int64_t d_out, int64_t p, int dtype, void* stream);

/* bca_fwd_spectral / bca_bwd_spectral — the layer with SPECTRAL-RESIDENT weights
 * (the paper keeps c's spectrum between steps, and its
 * training updates it in place: spectral-domain SGD with rdfft_packed_axpy):
 *   W:  fp32 [q_out][q_in][p] packed spectra W_ij = rdFFT(w_ij) (e.g. rdfft_fwd
 *       of an fp32 copy of w), read only; the kernels skip their weight transform.
 *   bca_fwd_spectral:  y = IrdFFT(sum_j W_ij (.) X_j)  (accumulate != 0: y += ...)
 *   bca_bwd_spectral:  dx as bca_bwd (dx may alias g iff d_in == d_out), and
 *       dW = sum_t conj(X_tj) (.) G_ti as fp32 PACKED SPECTRA, no inverse (accumulate
 *       != 0: added to dW's contents).  dW is rdFFT(dL/dw), the rdFFT of the
 *       time-domain weight gradient: the update of spectral-domain SGD
 *       (W -= lr dW, rdfft_packed_axpy; identical to time-domain SGD on w).  It is
 *       NOT dL/dW — the packed slots of W are not independent coordinates of w;
 *       dL/dW would weight slots 0 and p/2 by 1/p and every other slot by 2/p.
 *   Other arguments, layouts and errors as bca_fwd / bca_bwd.                 */
int bca_fwd_spectral(const void* x, const float* W, void* y, int64_t T, int64_t d_in, int64_t d_out, int64_t p,
                     int dtype, int accumulate, void* stream);
int bca_bwd_spectral(const void* x, const float* W, const void* g, void* dx, float* dW, int64_t T, int64_t d_in,
                     int64_t d_out, int64_t p, int dtype, int accumulate, void* stream);

/* ---- packed-spectrum utilities ---------------------------
 * rdfft_decode — the explicit decode step of the paper's Limitations
 * ("explicit complex access needs a decode step that breaks the
 * in-place property").  Out of place:
 *   p: [batch][n] packed spectra (read only)
 *   c: [batch][n + 2] interleaved bins (Re y_k, Im y_k), k = 0 .. n/2 — the
 *      torch.fft.rfft layout; Im y_0 = Im y_{n/2} = 0 are written explicitly.
 *   c may not overlap p (RDFFT_E_ALIAS).  Exact (a permutation).            */
int rdfft_decode(const void* p, void* c, int64_t batch, int64_t n, int dtype, void* stream);

/* rdfft_encode — inverse of rdfft_decode: c [batch][n + 2] -> p [batch][n]
 * packed.  Im y_0 and Im y_{n/2} are ignored (zero for the
 * spectrum of a real signal, Thm 1; not checked).  No overlap.   */
int rdfft_encode(const void* c, void* p, int64_t batch, int64_t n, int dtype, void* stream);

/* rdfft_packed_conj — a <- conj(a) per bin, in place (the conjugate of a
 * Hermitian spectrum stays Hermitian): slots n/2+1 .. n-1 (the
 * imaginary parts) change sign; exact.                              */
int rdfft_packed_conj(void* a, int64_t batch, int64_t n, int dtype, void* stream);

/* rdfft_packed_axpy — y <- y + alpha x, in the packed domain (the packing is
 * linear, so this is the spectral axpy; alpha = -lr gives a spectral-domain
 * SGD step).  y: [batch][n] in/out; x: [x_batch][n] read only,
 * x_batch == 1 broadcasts.  fp32 FMA; bf16 results rounded to nearest even.
 * x may not overlap y unless x == y and x_batch == batch.                   */
int rdfft_packed_axpy(void* y, const void* x, float alpha, int64_t batch, int64_t n, int64_t x_batch, int dtype,
                      void* stream);

/* Static, never-allocating description of a status code. */
const char* rdfft_status_str(int status);

/* rdfft_filter_host — the transform path end to end from HOST memory: every
 * row of xh becomes IrdFFT(rdFFT(row) (.) filt) (filt = NULL: the plain round
 * trip IrdFFT(rdFFT(row)); conj != 0: (.) conj(filt)), the circular
 * convolution of the row with the filter's impulse response (P:L165-172 with
 * one block; P:L290-293 for the product).
 *   xh:     HOST [batch][n] in/out.  Pinned (cudaHostAlloc / torch pin_memory)
 *           for the copies to overlap the kernels; pageable memory is correct
 *           but serialises.
 *   filt:   DEVICE [n] packed spectrum (one row, broadcast), or NULL.
 *   work:   DEVICE buffer of work_rows rows of n elements (caller-owned
 *           workspace, work_rows >= 2): two halves that alternate between
 *           stream0 and stream1.
 *   Chunk c of at most work_rows/2 rows runs on stream (c % 2) through half
 *   (c % 2): cudaMemcpyAsync host -> device, rdfft_fwd, rdfft_packed_mul
 *   (if filt), rdfft_inv, cudaMemcpyAsync device -> host.  Consecutive chunks
 *   on the two streams overlap their copies (both PCIe directions) with the
 *   other chunk's kernels; the same half is reused only in its own stream's
 *   order, so no event is needed.  Asynchronous: xh holds the result once both
 *   streams have drained (the caller synchronises them; the streams must
 *   already be ordered after the caller's earlier work on xh / filt / work).
 *   stream0 == stream1 is allowed (no overlap).  No allocation.
 *   Errors: as rdfft_fwd / rdfft_packed_mul, E_SHAPE for work_rows < 2,
 *   E_ALIAS if filt overlaps work, E_CUDA if a copy cannot be enqueued.      */
int rdfft_filter_host(void* xh, int64_t batch, int64_t n, int dtype, const void* filt, int conj, void* work,
                      int64_t work_rows, void* stream0, void* stream1);

/* Number of kernels this library has launched since load (process-wide,
 * monotonically increasing).  Used by bench.py to count its GPU launches.   */
uint64_t rdfft_launch_count(void);

/* Library ABI version (major*100 + minor). */
int rdfft_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RDFFT_H */
