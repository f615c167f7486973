// fast.h — declarations of the specialised launchers, each explicitly instantiated in its
// own translation unit (tu_*.cu) so the library compiles in parallel.  Host-only interface.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rdfft {
// plan3.cuh: specialised rdFFT kernels for every n in [2, 4096]; false if none applies.
template <typename T>
bool launch_rdfft_fast(T* x, int64_t batch, int n, int logn, bool inverse, int sms, cudaStream_t st);
// bca2.cuh: fused BCA fast paths (square layers, q <= 4, p in {256, 512, 1024}).
template <typename T>
bool bca_fwd_fast(const T* x, const T* w, T* y, int64_t T_, int q_in, int q_out, int p, int sms, cudaStream_t st,
                  int acc, const float* wspec);  // acc != 0: y += BCA(x); wspec: resident W spectra (else w)
template <typename T>
bool bca_bwd_fast(const T* x, const T* w, const T* g, T* dx, float* dw, int64_t T_, int q_in, int q_out, int p,
                  int sms, cudaStream_t st, const float* wspec);
// utils.cu: packed-spectrum utilities
template <typename T>
void launch_packed_conj(T* a, int64_t batch, int n, int logn, int sms, cudaStream_t st);
template <typename T>
void launch_packed_axpy(T* y, const T* x, float alpha, int64_t batch, int n, bool bcast, int sms, cudaStream_t st);
template <typename T>
void launch_decode(const T* p, T* c, int64_t batch, int n, int sms, cudaStream_t st);
template <typename T>
void launch_encode(const T* c, T* p, int64_t batch, int n, int sms, cudaStream_t st);
template <typename T>
void launch_packed_mul_large(T* a, const T* b, int64_t batch, int n, bool bcast, bool conj, int sms, cudaStream_t st);
}  // namespace rdfft
