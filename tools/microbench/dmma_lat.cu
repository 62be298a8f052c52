// DMMA.8x8x4 latency / single-warp throughput: 1 warp per SM, CH independent accumulator chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double d0[CH], d1[CH];
  for (int i = 0; i < CH; ++i) { d0[i] = 0; d1[i] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0[i]), "+d"(d1[i]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < CH; ++i) s += d0[i] + d1[i];
  out[blockIdx.x * 32 + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH> void run(double* out, long long* dc, int warps) {
  int iters = 2000;
  k<CH><<<1, 32 * warps>>>(out, dc, 10); cudaDeviceSynchronize();
  k<CH><<<1, 32 * warps>>>(out, dc, iters); cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("{\"test\":\"dmma_lat\",\"chains\":%d,\"warps\":%d,\"clk_per_dmma_per_warp\":%.2f}\n", CH, warps, (double)c / (iters * CH));
}
int main() { double* out; long long* dc; cudaMalloc(&out, 1 << 20); cudaMalloc(&dc, 8);
  run<1>(out, dc, 1); run<2>(out, dc, 1); run<4>(out, dc, 1); run<8>(out, dc, 1);
  run<1>(out, dc, 4); run<2>(out, dc, 4); run<4>(out, dc, 4); run<1>(out, dc, 16); run<2>(out, dc, 16);
  return 0; }
