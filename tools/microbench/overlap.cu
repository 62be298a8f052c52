// Is DMMA.8x8x4 with destination D overlapping source A (or B) correct on sm_100a?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, const double* in, int mode) {
  const int lane = threadIdx.x & 31;
  double a = in[lane], b = in[32 + lane];
  double d0, d1;
  if (mode == 0) {           // no overlap: D fresh, C = 0
    d0 = 0; d1 = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  } else if (mode == 1) {    // D0 tied to A
    double x = a, y = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%0}, {%2}, {%3,%3};\n" : "+d"(x), "=d"(y) : "d"(b), "d"(0.0));
    d0 = x; d1 = y;
  } else {                   // D0 tied to B
    double x = b, y = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%0}, {%3,%3};\n" : "+d"(x), "=d"(y) : "d"(a), "d"(0.0));
    d0 = x; d1 = y;
  }
  out[lane * 2] = d0; out[lane * 2 + 1] = d1;
}
int main() {
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 0.25 + 0.125 * i - 0.001 * i * i;
  double *in, *out; cudaMalloc(&in, 64 * 8); cudaMalloc(&out, 64 * 8);
  cudaMemcpy(in, h, 64 * 8, cudaMemcpyHostToDevice);
  double r[3][64];
  for (int m = 0; m < 3; ++m) { k<<<1, 32>>>(out, in, m); cudaMemcpy(r[m], out, 64 * 8, cudaMemcpyDeviceToHost); }
  int bad1 = 0, bad2 = 0; for (int i = 0; i < 64; ++i) { bad1 += r[1][i] != r[0][i]; bad2 += r[2][i] != r[0][i]; }
  printf("overlap D=A mismatches %d, D=B mismatches %d (of 64); sample %g %g %g\n", bad1, bad2, r[0][5], r[1][5], r[2][5]);
  return 0;
}
