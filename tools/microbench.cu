// tools/microbench.cu -- measured B200 co-bounds for the roofline:
//   1. FP64 FMA throughput (independent DFMA chains);
//   2. HBM read+write bandwidth of a gather/scatter copy whose contiguous
//      runs are 2^L amplitudes (16 B each), L = 0..6, at 4 GiB.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench.cu -o tools/microbench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fma_chain(double *out, int iters, double a, double b)
{
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1234.5) out[0] = x0;
}

// element i of the copy: run r = i >> L, offset o = i & (2^L-1); runs are
// scattered with stride 2^(L+S) so that consecutive runs are far apart
__global__ void gather_copy(const double2 *__restrict__ in, double2 *__restrict__ out, uint64_t n, int L, int S,
                            int lgN)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        // rotate the run index so that runs are visited in a strided order
        const uint64_t r = i >> L, o = i & ((1ull << L) - 1);
        const int rb = lgN - L;
        const uint64_t rr = ((r << S) | (r >> (rb - S))) & ((1ull << rb) - 1);
        const uint64_t j = (rr << L) | o;
        out[j] = in[j];
    }
}

int main()
{
    double *d;
    cudaMalloc(&d, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    fma_chain<<<sms * 8, 256>>>(d, 16, 1.0000001, 1e-9);
    cudaEventRecord(a);
    fma_chain<<<sms * 8, 256>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fmas = (double)sms * 8 * 256 * iters * 64;
    printf("{\"fp64_fma_per_s\": %.4e, \"fp64_tflops\": %.3f, \"fma_per_clk_per_sm_at_max\": %.1f}\n", fmas / (ms * 1e-3),
           2 * fmas / (ms * 1e-3) / 1e12, fmas / (ms * 1e-3) / sms / 1.965e9);
    const int lgN = 28;
    const uint64_t n = 1ull << lgN;
    double2 *x, *y;
    cudaMalloc(&x, n * 16);
    cudaMalloc(&y, n * 16);
    cudaMemset(x, 0, n * 16);
    for (int L = 0; L <= 6; ++L) {
        gather_copy<<<sms * 16, 256>>>(x, y, n, L, 9, lgN);
        cudaEventRecord(a);
        for (int rep = 0; rep < 5; ++rep) gather_copy<<<sms * 16, 256>>>(x, y, n, L, 9, lgN);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"run_bytes\": %d, \"copy_gbs\": %.1f}\n", 16 << L, 5.0 * n * 32 / (ms * 1e-3) / 1e9);
    }
    return 0;
}
