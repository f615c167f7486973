// Does FFMA2 free issue slots for co-issued ALU / LDS work? (B200 sm_100a)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float2 v){unsigned long long r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(v.x),"f"(v.y)); return r;}
__device__ __forceinline__ float2 u2f(unsigned long long r){float2 v; asm("mov.b64 {%0,%1}, %2;":"=f"(v.x),"=f"(v.y):"l"(r)); return v;}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c){ unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(d):"l"(f2u(a)),"l"(f2u(b)),"l"(f2u(c))); return u2f(d);}
template<int MODE>
__global__ void k(float* out, int iters, float a, float b) {
  a += threadIdx.x*1e-9f; b += threadIdx.x*1e-9f;
  float2 A=make_float2(a,a), B=make_float2(b,b);
  float2 x[8]; for(int j=0;j<8;j++) x[j]=make_float2(threadIdx.x+j, threadIdx.x-j);
  float y[8]; for(int j=0;j<8;j++) y[j]=threadIdx.x*0.5f+j;
  unsigned u[8]; for(int j=0;j<8;j++) u[j]=threadIdx.x*7+j;
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int q=0;q<8;q++){
      if (MODE==0 || MODE==2 || MODE==4) x[q]=fma2(x[q],A,B);
      if (MODE==1 || MODE==2) { asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[q]) : "r"(u[(q+1)&7]), "r"(u[(q+2)&7])); }
      if (MODE==3 || MODE==4) { y[q]=fmaf(y[q],a,b); }
      if (MODE==5) { y[q]=fmaf(y[q],a,b); asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[q]) : "r"(u[(q+1)&7]), "r"(u[(q+2)&7])); }
    } }
  float s=0; for(int j=0;j<8;j++) s+=x[j].x+x[j].y+y[j]+(float)u[j];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float* out; cudaMalloc(&out, 148*8*256*4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks=148*8, thr=256, iters=4000; float ms;
  const char* names[]={"FFMA2 only","LOP3 only","FFMA2+LOP3","FFMA only","FFMA2+FFMA","FFMA+LOP3"};
  for(int rep=0;rep<2;rep++) for(int m=0;m<6;m++){
    cudaEventRecord(e0);
    switch(m){case 0:k<0><<<blocks,thr>>>(out,iters,.999f,.001f);break;case 1:k<1><<<blocks,thr>>>(out,iters,.999f,.001f);break;
      case 2:k<2><<<blocks,thr>>>(out,iters,.999f,.001f);break;case 3:k<3><<<blocks,thr>>>(out,iters,.999f,.001f);break;
      case 4:k<4><<<blocks,thr>>>(out,iters,.999f,.001f);break;case 5:k<5><<<blocks,thr>>>(out,iters,.999f,.001f);break;}
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
    double w=(double)blocks*thr/32*iters*8; // warp-iterations of the 8-op body
    if(rep) printf("%-12s: %.3f ms  -> %.2f cycles per (warp, op-slot) at 1.965GHz per SMSP\n", names[m], ms, ms*1e-3*1.965e9*148*4/w);
  }
  return 0;
}
