// Microbenchmark: throughput of shared -> global bulk copies (cp.async.bulk, the
// TMA engine's non-tensor copy; UBLKCP in SASS) as a function of the copy size,
// against warp-cooperative 16-byte streaming stores of the same bytes.
//
// Each warp owns a 10 KB shared staging buffer and streams `bytes`-sized segments to
// consecutive destinations of a 4 GB output (larger than L2), as the Gram write-out
// does: lanes 0..R-1 each issue one copy per round (R = rows per round, 8 in v3).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulkcopy bulkcopy.cu && ./bulkcopy
// prints one JSON line per (mode, bytes): GB/s and SM cycles per copy per SM.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int WARPS = 4;

__global__ void __launch_bounds__(WARPS * 32) bulk_kernel(double *out, long long n_seg, int bytes, int rows, int mode)
{
    __shared__ __align__(128) double stage[WARPS][1280];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = lane; i < 1280; i += 32) stage[warp][i] = i;
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    const long long gw = (long long)blockIdx.x * WARPS + warp, nw = (long long)gridDim.x * WARPS;
    const int dbl = bytes / 8;
    for (long long s0 = gw * rows; s0 < n_seg; s0 += nw * rows) {
        if (mode == 0) {  // bulk copies, one per lane < rows
            if (lane < rows && s0 + lane < n_seg) {
                double *dst = out + (s0 + lane) * dbl;
                const unsigned src = (unsigned)__cvta_generic_to_shared(&stage[warp][(lane * dbl) & 255]);
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(src),
                             "r"(bytes) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            __syncwarp();
        } else {  // the warp stores the rows itself, 16 bytes per lane per instruction
            for (int r = 0; r < rows && s0 + r < n_seg; ++r) {
                double2 *dst = reinterpret_cast<double2 *>(out + (s0 + r) * dbl);
                const double2 *src = reinterpret_cast<const double2 *>(&stage[warp][(r * dbl) & 255]);
                for (int c = lane; c < dbl / 2; c += 32) __stcs(dst + c, src[c]);
            }
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int main()
{
    const size_t total = 4ull << 30;
    double *out;
    CK(cudaMalloc(&out, total));
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int sizes[] = {128, 256, 400, 512, 800, 1024, 2048, 4096, 8192};
    for (int mode = 0; mode < 2; ++mode)
        for (int bytes : sizes) {
            const long long n_seg = (long long)(total / bytes);
            const int grid = sms * 8;
            bulk_kernel<<<grid, WARPS * 32>>>(out, n_seg, bytes, 8, mode);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            bulk_kernel<<<grid, WARPS * 32>>>(out, n_seg, bytes, 8, mode);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double gbs = (double)n_seg * bytes / (ms * 1e-3) / 1e9;
            const double cyc = (ms * 1e-3) * clk * 1e3 / ((double)n_seg / sms);
            printf("{\"test\":\"%s\",\"bytes\":%d,\"gbs\":%.1f,\"sm_cycles_per_segment\":%.2f}\n",
                   mode == 0 ? "bulk_copy" : "warp_stcs16", bytes, gbs, cyc);
        }
    return 0;
}
