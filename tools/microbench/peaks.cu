// Microbenchmarks for the FP64 roofline denominators on B200 (sm_100a):
// DFMA chain throughput, DMMA (mma.sync f64) throughput, write-only HBM BW.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b){
  double acc[CH];
  #pragma unroll
  for(int i=0;i<CH;i++) acc[i]=threadIdx.x*1e-3+i;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CH;i++) acc[i]=fma(acc[i],a,b);
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<CH;i++) s+=acc[i];
  if(s==12345.678) out[threadIdx.x]=s;
}

template<int CH>
__global__ void dmma_kernel(double* out, int iters){
  double a = 1.0 + threadIdx.x*1e-9, b = 0.5 - threadIdx.x*1e-9;
  double c0[CH], c1[CH];
  #pragma unroll
  for(int i=0;i<CH;i++){c0[i]=0;c1[i]=0;}
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CH;i++){
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
    }
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<CH;i++) s+=c0[i]+c1[i];
  if(s==12345.678) out[threadIdx.x]=s;
}

template<int CH>
__global__ void dmma16_kernel(double* out, int iters){
  double a0 = 1.0 + threadIdx.x*1e-9, a1=a0*0.5, b = 0.5 - threadIdx.x*1e-9;
  double c[CH][4];
  #pragma unroll
  for(int i=0;i<CH;i++){c[i][0]=c[i][1]=c[i][2]=c[i][3]=0;}
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CH;i++){
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<CH;i++) s+=c[i][0]+c[i][1]+c[i][2]+c[i][3];
  if(s==12345.678) out[threadIdx.x]=s;
}

__global__ void write_kernel(double2* __restrict__ p, size_t n2){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x*blockDim.x;
  double2 v = make_double2(1.0, 2.0);
  for(; i<n2; i+=stride) p[i]=v;
}
__global__ void write_cs_kernel(double2* __restrict__ p, size_t n2){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x*blockDim.x;
  double2 v = make_double2(1.0, 2.0);
  for(; i<n2; i+=stride) __stcs(p+i, v);
}

int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,dev));
  int sms=pr.multiProcessorCount;
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d}\n", pr.name, sms, clk);
  double* out; CK(cudaMalloc(&out, 1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  for(int bs: {256, 512, 1024}){
    int iters=20000; int grid=sms*(2048/bs);
    dfma_kernel<8><<<grid,bs>>>(out,100,1.0000001,1e-9); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_kernel<8><<<grid,bs>>>(out,iters,1.0000001,1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*8*iters*(double)grid*bs;
    printf("{\"test\":\"dfma\",\"block\":%d,\"grid\":%d,\"tflops\":%.3f}\n", bs, grid, fl/ms/1e9);
  }
  // DMMA m8n8k4
  for(int bs: {128, 256, 512}){
    int iters=4000; int grid=sms*(1024/bs);
    dmma_kernel<4><<<grid,bs>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_kernel<4><<<grid,bs>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*256*4*iters*(double)grid*(bs/32);
    printf("{\"test\":\"dmma_m8n8k4\",\"block\":%d,\"grid\":%d,\"tflops\":%.3f}\n", bs, grid, fl/ms/1e9);
  }
  for(int bs: {128, 256}){
    int iters=4000; int grid=sms*(1024/bs);
    dmma16_kernel<4><<<grid,bs>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma16_kernel<4><<<grid,bs>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*512*4*iters*(double)grid*(bs/32);
    printf("{\"test\":\"dmma_m16n8k4\",\"block\":%d,\"grid\":%d,\"tflops\":%.3f}\n", bs, grid, fl/ms/1e9);
  }
  // write-only BW
  size_t bytes = (size_t)8<<30; double2* buf; CK(cudaMalloc(&buf, bytes));
  size_t n2 = bytes/16;
  for(int mode=0; mode<3; ++mode){
    for(int w=0; w<2; ++w){ if(mode==0) write_kernel<<<sms*8,256>>>(buf,n2); else if(mode==1) write_cs_kernel<<<sms*8,256>>>(buf,n2); else cudaMemsetAsync(buf,0,bytes);} 
    CK(cudaDeviceSynchronize());
    float best=1e9;
    for(int r=0;r<5;r++){
      cudaEventRecord(e0);
      if(mode==0) write_kernel<<<sms*8,256>>>(buf,n2); else if(mode==1) write_cs_kernel<<<sms*8,256>>>(buf,n2); else cudaMemsetAsync(buf,0,bytes);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); if(ms<best) best=ms;
    }
    const char* nm[3]={"write_stg128","write_stcs128","memset"};
    printf("{\"test\":\"%s\",\"gbs\":%.1f}\n", nm[mode], bytes/best/1e6);
  }
  return 0;
}
