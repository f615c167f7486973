// synccheck_tmem.cu — does compute-sanitizer --tool synccheck accept a CTA that allocates tensor memory
// (tcgen05.alloc / tcgen05.st / tcgen05.ld / dealloc) with named barriers but no mbarrier?
//   kernel 0: TMEM alloc + st/ld + named barriers, no mbarrier
//   kernel 1: the same plus one initialised (unused) mbarrier
//   kernel 2: the same as 0 with a bar.arrive / bar.sync producer-consumer pair (bca_bwd4's pattern)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/sct synccheck_tmem.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(float* out) {
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  if (MODE == 1 && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = slot + ((uint32_t)(32 * ((tid / 32) % 4)) << 16) + (uint32_t)(16 * (tid / 128));
  uint32_t v = tid;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t), "r"(v) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (MODE == 2) {
    if (tid < 128) asm volatile("bar.arrive 3, 256;" ::: "memory");
    else asm volatile("bar.sync 3, 256;" ::: "memory");
  } else {
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
  out[blockIdx.x * 256 + tid] = (float)r;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot) : "memory");
}

int main(int argc, char** argv) {  // argv[1]: the mode to run (one per process: a failure is sticky)
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  float* out;
  cudaMalloc(&out, 4 * 256 * 4);
  if (mode == 0) k<0><<<4, 256>>>(out);
  if (mode == 1) k<1><<<4, 256>>>(out);
  if (mode == 2) k<2><<<4, 256>>>(out);
  printf("mode %d: %s\n", mode, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
