// Feasibility probe for L2-resident pass pairs: two streaming
// "passes" over a 4 GiB state, (a) each over the whole state (2 full HBM
// read+write sweeps), (b) chunked: pass A reads chunk c of X (HBM) and writes
// it to Y, pass B reads Y (L2) and writes X, chunk by chunk, optionally
// discarding Y's lines from L2 after B has read them (no write-back).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2_chunk_probe.cu -o /tmp/l2probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void pass_copy(const double2 *__restrict__ in, double2 *__restrict__ out, size_t n, double s, int discard)
{
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double2 v = in[i];
        out[i] = make_double2(v.x * s, v.y * s);
    }
    if (discard) {
        // every 128-byte line of `in` (8 double2), after the whole block has read it
        __syncthreads();
        for (size_t l = (size_t)blockIdx.x * blockDim.x + threadIdx.x; l < n / 8; l += stride)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(in + 8 * l) : "memory");
    }
}
int main()
{
    const size_t N = (size_t)1 << 28;   // 4 GiB of double2
    double2 *X, *Y;
    cudaMalloc(&X, N * 16);
    cudaMalloc(&Y, N * 16);
    cudaMemset(X, 0, N * 16);
    cudaMemset(Y, 0, N * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int g = 148 * 8, t = 256;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        pass_copy<<<g, t>>>(X, Y, N, 1.0, 0);
        pass_copy<<<g, t>>>(Y, X, N, 1.0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"mode\": \"two full passes\", \"ms\": %.3f}\n", ms);
    }
    for (size_t chunk_mb : {8, 16, 32, 64}) {
        for (int disc = 0; disc < 2; ++disc) {
            const size_t C = chunk_mb * (1 << 20) / 16;
            cudaEventRecord(a);
            for (size_t c = 0; c < N; c += C) {
                pass_copy<<<g, t>>>(X + c, Y + c, C, 1.0, 0);
                pass_copy<<<g, t>>>(Y + c, X + c, C, 1.0, disc);
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("{\"mode\": \"chunked\", \"chunk_mb\": %zu, \"discard\": %d, \"ms\": %.3f}\n", chunk_mb, disc, ms);
        }
    }
    // per-kernel times inside the chunked loop (32 MiB chunks)
    {
        const size_t C = (size_t)32 * (1 << 20) / 16;
        cudaEvent_t e[4];
        for (auto &x : e) cudaEventCreate(&x);
        for (size_t c = 0; c < N; c += C) {
            const bool probe = c == N / 2;
            if (probe) cudaEventRecord(e[0]);
            pass_copy<<<g, t>>>(X + c, Y + c, C, 1.0, 0);
            if (probe) cudaEventRecord(e[1]);
            pass_copy<<<g, t>>>(Y + c, X + c, C, 1.0, 0);
            if (probe) cudaEventRecord(e[2]);
        }
        cudaDeviceSynchronize();
        float m1, m2;
        cudaEventElapsedTime(&m1, e[0], e[1]);
        cudaEventElapsedTime(&m2, e[1], e[2]);
        printf("{\"mode\": \"per-kernel 32MiB\", \"passA_us\": %.1f, \"passB_us\": %.1f, \"passA_TBps\": %.2f, \"passB_TBps\": %.2f}\n",
               m1 * 1e3, m2 * 1e3, 2 * 32.0 * (1 << 20) / (m1 * 1e-3) / 1e12, 2 * 32.0 * (1 << 20) / (m2 * 1e-3) / 1e12);
    }
    return 0;
}
