// tools/ops_ideal.cu -- measurement only: FP64 efficiency of dense 2x2 pair
// updates on 32 register-resident amplitudes per thread, 8 warps per SM,
// without the gate-list interpreter (op = dense 2x2 on window bit i % 5,
// matrices from shared memory): the ceiling the k_ops_* kernels can reach.
// VAR 0: plain C pair update; VAR 1: 4-way split accumulation (shallower chains)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Op { double2 u[4]; };

template <int B, int VAR>
__device__ __forceinline__ void dense(double2 (&v)[32], const double2 u0, const double2 u1, const double2 u2, const double2 u3)
{
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if (k & (1 << B)) continue;
        const double2 x = v[k], y = v[k | (1 << B)];
        if (VAR == 0) {
            v[k] = make_double2(fma(u0.x, x.x, fma(-u0.y, x.y, fma(u1.x, y.x, -u1.y * y.y))),
                                fma(u0.x, x.y, fma(u0.y, x.x, fma(u1.x, y.y, u1.y * y.x))));
            v[k | (1 << B)] = make_double2(fma(u2.x, x.x, fma(-u2.y, x.y, fma(u3.x, y.x, -u3.y * y.y))),
                                           fma(u2.x, x.y, fma(u2.y, x.x, fma(u3.x, y.y, u3.y * y.x))));
        } else {
            const double a = fma(u0.x, x.x, -u0.y * x.y), b = fma(u1.x, y.x, -u1.y * y.y);
            const double c = fma(u0.x, x.y, u0.y * x.x), d = fma(u1.x, y.y, u1.y * y.x);
            const double e = fma(u2.x, x.x, -u2.y * x.y), f = fma(u3.x, y.x, -u3.y * y.y);
            const double g = fma(u2.x, x.y, u2.y * x.x), hh = fma(u3.x, y.y, u3.y * y.x);
            v[k] = make_double2(a + b, c + d);
            v[k | (1 << B)] = make_double2(e + f, g + hh);
        }
    }
}

// 16 amplitudes per thread, 512 threads (16 warps per SM)
template <int B>
__device__ __forceinline__ void dense16(double2 (&v)[16], const double2 u0, const double2 u1, const double2 u2, const double2 u3)
{
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k & (1 << B)) continue;
        const double2 x = v[k], y = v[k | (1 << B)];
        v[k] = make_double2(fma(u0.x, x.x, fma(-u0.y, x.y, fma(u1.x, y.x, -u1.y * y.y))),
                            fma(u0.x, x.y, fma(u0.y, x.x, fma(u1.x, y.y, u1.y * y.x))));
        v[k | (1 << B)] = make_double2(fma(u2.x, x.x, fma(-u2.y, x.y, fma(u3.x, y.x, -u3.y * y.y))),
                                       fma(u2.x, x.y, fma(u2.y, x.x, fma(u3.x, y.y, u3.y * y.x))));
    }
}

__global__ void __launch_bounds__(512, 1) k_ideal16(double2 *psi, const Op *ops_g, int nops, uint64_t ntiles)
{
    __shared__ Op ops[64];
    for (int i = threadIdx.x; i < nops; i += blockDim.x) ops[i] = ops_g[i];
    __syncthreads();
    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        double2 v[16];
        double2 *base = psi + T * 8192 + threadIdx.x;
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = base[512 * k];
        for (int i = 0; i < nops; ++i) {
            const double2 u0 = ops[i].u[0], u1 = ops[i].u[1], u2 = ops[i].u[2], u3 = ops[i].u[3];
            switch (i % 4) {
            case 0: dense16<0>(v, u0, u1, u2, u3); break;
            case 1: dense16<1>(v, u0, u1, u2, u3); break;
            case 2: dense16<2>(v, u0, u1, u2, u3); break;
            default: dense16<3>(v, u0, u1, u2, u3); break;
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) base[512 * k] = v[k];
    }
}

template <int VAR>
__global__ void __launch_bounds__(256, 1) k_ideal(double2 *psi, const Op *ops_g, int nops, uint64_t ntiles)
{
    __shared__ Op ops[64];
    for (int i = threadIdx.x; i < nops; i += blockDim.x) ops[i] = ops_g[i];
    __syncthreads();
    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        double2 v[32];
        double2 *base = psi + T * 8192 + threadIdx.x;
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = base[256 * k];
        for (int i = 0; i < nops; ++i) {
            const double2 u0 = ops[i].u[0], u1 = ops[i].u[1], u2 = ops[i].u[2], u3 = ops[i].u[3];
            switch (i % 5) {
            case 0: dense<0, VAR>(v, u0, u1, u2, u3); break;
            case 1: dense<1, VAR>(v, u0, u1, u2, u3); break;
            case 2: dense<2, VAR>(v, u0, u1, u2, u3); break;
            case 3: dense<3, VAR>(v, u0, u1, u2, u3); break;
            default: dense<4, VAR>(v, u0, u1, u2, u3); break;
            }
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) base[256 * k] = v[k];
    }
}


// DENSE2-like op: two matrices selected by window bit C
template <int B, int C>
__device__ __forceinline__ void dense2(double2 (&v)[32], const double2 *u)
{
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if (k & (1 << B)) continue;
        const double2 *m = ((k >> C) & 1) ? u + 4 : u;
        const double2 u0 = m[0], u1 = m[1], u2 = m[2], u3 = m[3];
        const double2 x = v[k], y = v[k | (1 << B)];
        v[k] = make_double2(fma(u0.x, x.x, fma(-u0.y, x.y, fma(u1.x, y.x, -u1.y * y.y))),
                            fma(u0.x, x.y, fma(u0.y, x.x, fma(u1.x, y.y, u1.y * y.x))));
        v[k | (1 << B)] = make_double2(fma(u2.x, x.x, fma(-u2.y, x.y, fma(u3.x, y.x, -u3.y * y.y))),
                                       fma(u2.x, x.y, fma(u2.y, x.x, fma(u3.x, y.y, u3.y * y.x))));
    }
}

struct Op8 { double2 u[8]; };

// TR: a shared-memory transpose (write all 32, barrier, read back permuted) every 7 ops
template <bool TR>
__global__ void __launch_bounds__(256, 1) k_ideal2(double2 *psi, const Op8 *ops_g, int nops, uint64_t ntiles)
{
    extern __shared__ double2 sh[];
    Op8 *ops = reinterpret_cast<Op8 *>(sh + 8192);
    for (int i = threadIdx.x; i < nops; i += blockDim.x) ops[i] = ops_g[i];
    __syncthreads();
    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        double2 v[32];
        double2 *base = psi + T * 8192 + threadIdx.x;
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = base[256 * k];
        for (int i = 0; i < nops; ++i) {
            const double2 *u = ops[i].u;
            switch (i % 5) {
            case 0: dense2<0, 1>(v, u); break;
            case 1: dense2<1, 2>(v, u); break;
            case 2: dense2<2, 3>(v, u); break;
            case 3: dense2<3, 4>(v, u); break;
            default: dense2<4, 0>(v, u); break;
            }
            if (TR && (i % 7) == 6) {
                __syncthreads();
#pragma unroll
                for (int k = 0; k < 32; ++k) sh[(threadIdx.x * 32 + k) ^ (threadIdx.x & 7)] = v[k];
                __syncthreads();
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = sh[(threadIdx.x * 32 + k) ^ (threadIdx.x & 7)];
            }
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) base[256 * k] = v[k];
    }
}


// a dense 2x2 on lane bit L: each thread keeps its own row, the partner's
// amplitude arrives by shuffle (4 x 32-bit per double2)
__device__ __forceinline__ double shfl_d(double x, int m)
{
    int lo = __double2loint(x), hi = __double2hiint(x);
    lo = __shfl_xor_sync(0xffffffffu, lo, m);
    hi = __shfl_xor_sync(0xffffffffu, hi, m);
    return __hiloint2double(hi, lo);
}
template <int L>
__device__ __forceinline__ void dense_lane(double2 (&v)[32], const double2 u0, const double2 u1, const double2 u2,
                                           const double2 u3)
{
    const bool hi = (threadIdx.x >> L) & 1;
    const double2 a = hi ? u3 : u0, b = hi ? u2 : u1;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        const double2 x = v[k];
        const double2 y = make_double2(shfl_d(x.x, 1 << L), shfl_d(x.y, 1 << L));
        v[k] = make_double2(fma(a.x, x.x, fma(-a.y, x.y, fma(b.x, y.x, -b.y * y.y))),
                            fma(a.x, x.y, fma(a.y, x.x, fma(b.x, y.y, b.y * y.x))));
    }
}

__global__ void __launch_bounds__(256, 1) k_ideal_lane(double2 *psi, const Op *ops_g, int nops, uint64_t ntiles)
{
    __shared__ Op ops[64];
    for (int i = threadIdx.x; i < nops; i += blockDim.x) ops[i] = ops_g[i];
    __syncthreads();
    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        double2 v[32];
        double2 *base = psi + T * 8192 + threadIdx.x;
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = base[256 * k];
        for (int i = 0; i < nops; ++i) {
            const double2 u0 = ops[i].u[0], u1 = ops[i].u[1], u2 = ops[i].u[2], u3 = ops[i].u[3];
            switch (i % 9) {
            case 0: dense<0, 0>(v, u0, u1, u2, u3); break;
            case 1: dense<1, 0>(v, u0, u1, u2, u3); break;
            case 2: dense<2, 0>(v, u0, u1, u2, u3); break;
            case 3: dense<3, 0>(v, u0, u1, u2, u3); break;
            case 4: dense<4, 0>(v, u0, u1, u2, u3); break;
            case 5: dense_lane<0>(v, u0, u1, u2, u3); break;
            case 6: dense_lane<1>(v, u0, u1, u2, u3); break;
            case 7: dense_lane<2>(v, u0, u1, u2, u3); break;
            default: dense_lane<3>(v, u0, u1, u2, u3); break;
            }
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) base[256 * k] = v[k];
    }
}

int main()
{
    const int n = 28, nops = 26;
    const uint64_t N = 1ull << n;
    double2 *psi;
    Op *ops;
    cudaMalloc(&psi, N * 16);
    cudaMemset(psi, 0, N * 16);
    cudaMalloc(&ops, 64 * sizeof(Op));
    Op h[64];
    for (int i = 0; i < 64; ++i)
        for (int k = 0; k < 4; ++k) h[i].u[k] = make_double2(0.5 + 0.01 * k, 0.25 - 0.01 * i);
    cudaMemcpy(ops, h, sizeof h, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int var = 0; var < 3; ++var) {
        auto go = [&]() {
            if (var == 0) k_ideal<0><<<sms, 256>>>(psi, ops, nops, N >> 13);
            else if (var == 1) k_ideal<1><<<sms, 256>>>(psi, ops, nops, N >> 13);
            else k_ideal16<<<sms, 512>>>(psi, ops, nops, N >> 13);
        };
        go();
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) go();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 3;
        const double instr = (double)nops * 16 * (N / 2);   // FP64 instructions (16 per pair)
        printf("{\"var\": %d, \"ms\": %.3f, \"fp64_instr_per_s\": %.4e, \"frac_of_64_per_clk_at_1965\": %.3f, \"err\": \"%s\"}\n",
               var, ms, instr / (ms * 1e-3), instr / (ms * 1e-3) / (sms * 64.0 * 1.965e9),
               cudaGetErrorString(cudaGetLastError()));
    }
    {
        Op8 *ops8;
        cudaMalloc(&ops8, 64 * sizeof(Op8));
        Op8 h8[64];
        for (int i = 0; i < 64; ++i)
            for (int k = 0; k < 8; ++k) h8[i].u[k] = make_double2(0.5 + 0.01 * k, 0.25 - 0.01 * i);
        cudaMemcpy(ops8, h8, sizeof h8, cudaMemcpyHostToDevice);
        const size_t sm = 8192 * 16 + 64 * sizeof(Op8);
        cudaFuncSetAttribute(k_ideal2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(k_ideal2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int tr = 0; tr < 2; ++tr) {
            auto go = [&]() {
                if (tr) k_ideal2<true><<<sms, 256, sm>>>(psi, ops8, nops, N >> 13);
                else k_ideal2<false><<<sms, 256, sm>>>(psi, ops8, nops, N >> 13);
            };
            go();
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) go();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 3;
            const double instr = (double)nops * 16 * (N / 2);
            printf("{\"var\": \"dense2%s\", \"ms\": %.3f, \"frac_of_64_per_clk_at_1965\": %.3f, \"err\": \"%s\"}\n",
                   tr ? "+transpose" : "", ms, instr / (ms * 1e-3) / (sms * 64.0 * 1.965e9),
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    {
        k_ideal_lane<<<sms, 256>>>(psi, ops, nops, N >> 13);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) k_ideal_lane<<<sms, 256>>>(psi, ops, nops, N >> 13);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 3;
        const double instr = (double)nops * 16 * (N / 2);
        printf("{\"var\": \"reg+lane ops (5 of 9 in registers, 4 by shuffle)\", \"ms\": %.3f, \"frac_of_64_per_clk_at_1965\": %.3f, \"err\": \"%s\"}\n",
               ms, instr / (ms * 1e-3) / (sms * 64.0 * 1.965e9), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
