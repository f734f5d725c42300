// FP64 pipe on this B200: dependent-chain latency and throughput vs ILP / warps
// (nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_lat.cu -o tools/fp64_lat)
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void chain(double *out, int iters, double a, double b)
{
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * (double)ILP);
}
template <int ILP>
void run(int warps_per_sm)
{
    double *d;
    cudaMalloc(&d, 148 * 1024 * sizeof(double) * 2);
    const int iters = 4096;
    chain<ILP><<<148, 32 * warps_per_sm>>>(d, iters, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chain<ILP><<<148, 32 * warps_per_sm>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double cyc; cudaMemcpy(&cyc, d, sizeof(double), cudaMemcpyDeviceToHost);
    double fma_per_s = 148.0 * 32 * warps_per_sm * (double)iters * ILP / (ms * 1e-3);
    printf("{\"ilp\": %d, \"warps_per_sm\": %d, \"cycles_per_fma_per_thread\": %.2f, \"fma_per_s\": %.4g}\n", ILP, warps_per_sm, cyc, fma_per_s);
    cudaFree(d);
}
int main()
{
    for (int w : {1, 2, 4, 8, 16}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
    return 0;
}
