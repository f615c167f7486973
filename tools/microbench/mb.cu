// Microbenchmarks to size the rdFFT kernel design on B200 (sm_100a):
// FFMA vs FFMA2 (fma.rn.f32x2) issue throughput, LDS throughput, HBM copy.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void k_ffma(float* out, int iters, float a, float b) {
  a += threadIdx.x*1e-9f; b += threadIdx.x*1e-9f;
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<8;j++){ x0=fmaf(x0,a,b); x1=fmaf(x1,a,b); x2=fmaf(x2,a,b); x3=fmaf(x3,a,b);
      x4=fmaf(x4,a,b); x5=fmaf(x5,a,b); x6=fmaf(x6,a,b); x7=fmaf(x7,a,b);} }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__device__ __forceinline__ unsigned long long f2u(float2 v){unsigned long long r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(v.x),"f"(v.y)); return r;}
__device__ __forceinline__ float2 u2f(unsigned long long r){float2 v; asm("mov.b64 {%0,%1}, %2;":"=f"(v.x),"=f"(v.y):"l"(r)); return v;}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c){ unsigned long long d; asm("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(d):"l"(f2u(a)),"l"(f2u(b)),"l"(f2u(c))); return u2f(d);}
__device__ __forceinline__ float2 add2(float2 a, float2 b){ unsigned long long d; asm("add.rn.f32x2 %0, %1, %2;":"=l"(d):"l"(f2u(a)),"l"(f2u(b))); return u2f(d);}
__global__ void k_ffma2(float* out, int iters, float a, float b) {
  a += threadIdx.x*1e-9f; b += threadIdx.x*1e-9f;
  float2 A=make_float2(a,a), B=make_float2(b,b);
  float2 x[8]; for(int j=0;j<8;j++) x[j]=make_float2(threadIdx.x+j, threadIdx.x-j);
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<8;j++){
#pragma unroll
      for(int q=0;q<8;q++) x[q]=fma2(x[q],A,B);} }
  float s=0; for(int j=0;j<8;j++) s+=x[j].x+x[j].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_fadd2(float* out, int iters, float a, float b) {
  a += threadIdx.x*1e-9f;
  float2 A=make_float2(a,a);
  float2 x[8]; for(int j=0;j<8;j++) x[j]=make_float2(threadIdx.x+j, threadIdx.x-j);
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<8;j++){
#pragma unroll
      for(int q=0;q<8;q++) x[q]=add2(x[q],A);} }
  float s=0; for(int j=0;j<8;j++) s+=x[j].x+x[j].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_fadd(float* out, int iters, float a, float b) {
  a += threadIdx.x*1e-9f;
  float x[8]; for(int j=0;j<8;j++) x[j]=threadIdx.x+j;
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<8;j++){
#pragma unroll
      for(int q=0;q<8;q++) x[q]=x[q]+a;} }
  float s=0; for(int j=0;j<8;j++) s+=x[j];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_lds(float* out, int iters) {
  __shared__ float sm[4096];
  for(int i=threadIdx.x;i<4096;i+=blockDim.x) sm[i]=i;
  __syncthreads();
  float s=0; int idx=threadIdx.x;
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<16;j++){ s+=sm[(idx + j*32)&4095]; }
    idx = (idx+ (int)s) & 4095;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_lds128(float* out, int iters) {
  __shared__ float4 sm[1024];
  for(int i=threadIdx.x;i<1024;i+=blockDim.x) sm[i]=make_float4(i,i,i,i);
  __syncthreads();
  float s=0; int idx=threadIdx.x;
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<16;j++){ float4 v=sm[(idx + j*32)&1023]; s+=v.x+v.y+v.z+v.w; }
    idx = (idx+ (int)s) & 1023;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n; i+= (size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
__global__ void k_inplace(int4* a, size_t n) {
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n; i+= (size_t)gridDim.x*blockDim.x) { int4 v=a[i]; v.x+=1; a[i]=v; }
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("name %s SMs %d smemPerBlockOptin %zu smemPerSM %zu regsPerSM %d L2 %d clock %d kHz memclk %d kHz busw %d\n",
    p.name,p.multiProcessorCount,p.sharedMemPerBlockOptin,p.sharedMemPerMultiprocessor,p.regsPerMultiprocessor,p.l2CacheSize,p.clockRate,p.memoryClockRate,p.memoryBusWidth);
  float* out; CK(cudaMalloc(&out, 148*8*1024*4*4));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks=148*8, thr=256, iters=2000; float ms;
  for(int rep=0;rep<2;rep++){
  cudaEventRecord(e0); k_ffma<<<blocks,thr>>>(out,iters,0.999f,0.001f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
  double ops=(double)blocks*thr*iters*64; printf("FFMA  : %.1f G lane-inst/s (%.1f TFLOPs)\n", ops/ms/1e6, 2*ops/ms/1e9);
  cudaEventRecord(e0); k_ffma2<<<blocks,thr>>>(out,iters,0.999f,0.001f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
  printf("FFMA2 : %.1f G lane-inst/s (%.1f TFLOPs)\n", ops/ms/1e6, 4*ops/ms/1e9);
  cudaEventRecord(e0); k_fadd<<<blocks,thr>>>(out,iters,0.999f,0.001f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
  printf("FADD  : %.1f G lane-inst/s\n", ops/ms/1e6);
  cudaEventRecord(e0); k_fadd2<<<blocks,thr>>>(out,iters,0.999f,0.001f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
  printf("FADD2 : %.1f G lane-inst/s (%.1f G flops)\n", ops/ms/1e6, 2*ops/ms/1e6);
  cudaEventRecord(e0); k_lds<<<blocks,thr>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
  double lds=(double)blocks*thr*iters*16; printf("LDS32 : %.1f G lane-ld/s = %.1f TB/s\n", lds/ms/1e6, lds*4/ms/1e9);
  cudaEventRecord(e0); k_lds128<<<blocks,thr>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
  printf("LDS128: %.1f G lane-ld/s = %.1f TB/s\n", lds/ms/1e6, lds*16/ms/1e9);
  }
  size_t bytes=(size_t)4<<30; int4 *a,*b; CK(cudaMalloc(&a,bytes)); CK(cudaMalloc(&b,bytes)); cudaMemset(a,0,bytes); cudaMemset(b,0,bytes);
  size_t n=bytes/16;
  for(int g: {148*4, 148*8, 148*16, 148*32}) for(int rep=0;rep<3;rep++){
    cudaEventRecord(e0); k_copy<<<g,256>>>(a,b,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    if(rep==2) printf("copy grid %d: %.1f GB/s\n", g, 2.0*bytes/ms/1e6);
    cudaEventRecord(e0); k_inplace<<<g,256>>>(a,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    if(rep==2) printf("inplace rw grid %d: %.1f GB/s\n", g, 2.0*bytes/ms/1e6);
  }
  cudaEventRecord(e0); cudaMemcpyAsync(b,a,bytes,cudaMemcpyDeviceToDevice); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
  printf("memcpy D2D: %.1f GB/s\n", 2.0*bytes/ms/1e6);
  return 0;
}
