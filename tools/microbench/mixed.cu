// Does FP64 DFMA issue concurrently with DMMA (separate pipes) on B200?
#include <cstdio>
#include <cuda_runtime.h>
template<int CM, int CF>
__global__ void mixed(double* out, int iters){
  double a = 1.0 + threadIdx.x*1e-9, b = 0.5 - threadIdx.x*1e-9;
  double c0[CM>0?CM:1], c1[CM>0?CM:1], f[CF>0?CF:1];
  #pragma unroll
  for(int i=0;i<(CM>0?CM:1);i++){c0[i]=0;c1[i]=0;}
  #pragma unroll
  for(int i=0;i<(CF>0?CF:1);i++) f[i]=threadIdx.x*1e-3+i;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CM;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
    #pragma unroll
    for(int j=0;j<4;j++){
    #pragma unroll
    for(int i=0;i<CF;i++) f[i]=fma(f[i],1.0000001,1e-9);
    }
  }
  double s=0;
  for(int i=0;i<CM;i++) s+=c0[i]+c1[i];
  for(int i=0;i<CF;i++) s+=f[i];
  if(s==12345.678) out[threadIdx.x]=s;
}
template<int CM,int CF> void run(double* out, int sms){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=4000, bs=256, grid=sms*4;
  mixed<CM,CF><<<grid,bs>>>(out,10); cudaDeviceSynchronize();
  cudaEventRecord(e0); mixed<CM,CF><<<grid,bs>>>(out,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  double warps=(double)grid*bs/32;
  double fm=2.0*256*CM*iters*warps, ff=2.0*32*CF*4*iters*warps;
  printf("{\"test\":\"mixed\",\"dmma_per_iter\":%d,\"dfma_per_iter\":%d,\"ms\":%.3f,\"dmma_tflops\":%.2f,\"dfma_tflops\":%.2f,\"total\":%.2f}\n",CM,CF*4,ms,fm/ms/1e9,ff/ms/1e9,(fm+ff)/ms/1e9);
}
int main(){ double* out; cudaMalloc(&out,1<<20); int sms=148;
  run<4,0>(out,sms); run<0,8>(out,sms); run<4,8>(out,sms); run<4,4>(out,sms); run<2,8>(out,sms); run<4,16>(out,sms);
  return 0; }
