// tools/pass_pattern.cu -- measurement only: HBM copy bandwidth of the read
// pattern of a fused QFT pass whose active wires sit on the top positions
// (rows of 2^r contiguous amplitudes, 2^(12-r) rows per 4096-amplitude tile,
// row stride 2^(n-12+r) amplitudes), written back contiguously (block-move
// layout).  Variants: TMA tensor load into a 3-stage ring + bulk store (the
// k_qft_tma data path), and a register double-buffered LDG gather.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lcuda tools/pass_pattern.cu -o tools/pass_pattern
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

constexpr int N = 28;
constexpr int TB = 12;
constexpr uint32_t TILE_BYTES = 16u << TB;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
            smem_u32(b)),
        "r"(ph)
        : "memory");
}

// 3-D tensor: dim0 = run (2^r amps as 2^(r+1) doubles), dim1 = tile id (middle bits),
// dim2 = row (top 12 - r bits).  Box = [run, 1, rows].
__global__ void __launch_bounds__(256, 1) k_tma(const __grid_constant__ CUtensorMap in, double2 *out, int r,
                                                uint64_t ntiles)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    double2 *bufs = reinterpret_cast<double2 *>(sm);
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + 3 * TILE_BYTES);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 3; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto load = [&](uint64_t T, int s) {
        mbar_expect_tx(&full[s], TILE_BYTES);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(smem_u32(bufs + (size_t)s * 4096)),
            "l"((uint64_t)&in), "r"(0), "r"((int)T), "r"(0), "r"(smem_u32(&full[s]))
            : "memory");
    };
    if (threadIdx.x == 0)
        for (int q = 0; q < 2; ++q)
            if (blockIdx.x + q * gridDim.x < ntiles) load(blockIdx.x + q * gridDim.x, q);
    uint64_t j = 0;
    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x, ++j) {
        const int s = (int)(j % 3);
        mbar_wait(&full[s], (uint32_t)((j / 3) & 1));
        // touch the data (a real pass reads it into registers)
        double2 *b = bufs + (size_t)s * 4096;
        double2 v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = b[threadIdx.x + 256 * k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) b[threadIdx.x + 256 * k] = make_double2(v[k].x + 1.0, v[k].y);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + T * 4096),
                         "r"(smem_u32(b)), "r"(TILE_BYTES)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            const uint64_t Tn = T + 2ull * gridDim.x;
            if (Tn < ntiles) load(Tn, (int)((j + 2) % 3));
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// LDG gather: thread t of 256 loads amplitude k (0..15) of the tile at
// element e = t + 256 k: run offset e & (2^r - 1), row e >> r.  Next tile's
// loads are issued before the current tile is stored (registers double buffer).
__global__ void __launch_bounds__(256, 2) k_ldg(const double2 *__restrict__ in, double2 *__restrict__ out, int r,
                                                uint64_t ntiles)
{
    const int mid = N - TB;   // tile id bits
    auto addr = [&](uint64_t T, uint32_t e) -> uint64_t {
        const uint64_t off = e & ((1u << r) - 1);
        const uint64_t row = e >> r;
        return off | (T << r) | (row << (r + mid));
    };
    double2 a[16], b[16];
    uint64_t T = blockIdx.x;
    if (T >= ntiles) return;
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = __ldcs(in + addr(T, threadIdx.x + 256 * k));
    for (; T < ntiles; T += gridDim.x) {
        const uint64_t Tn = T + gridDim.x;
        if (Tn < ntiles) {
#pragma unroll
            for (int k = 0; k < 16; ++k) b[k] = __ldcs(in + addr(Tn, threadIdx.x + 256 * k));
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) __stcs(out + T * 4096 + threadIdx.x + 256 * k, make_double2(a[k].x + 1.0, a[k].y));
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = b[k];
    }
}

// 2^13-amplitude tiles landing as four 32 KiB quarters in a ring of 7 slots
// (the k_qft13 schedule): MODE 0 = next loads issued after a full-tile
// "transpose" through the tile's slots (as k_qft13), MODE 1 = right after the
// landing read (no transpose: the pipeline's upper bound)
template <int MODE>
__global__ void __launch_bounds__(256, 1) k_q13(const __grid_constant__ CUtensorMap in, double2 *out, uint64_t ntiles)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    double2 *slots = reinterpret_cast<double2 *>(sm);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 7 * 32768);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 7; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](uint64_t s) {
        const uint64_t T = blockIdx.x + (s >> 2) * gridDim.x;
        if (T >= ntiles) return;
        const int q = (int)(s & 3), sl = (int)(s % 7);
        mbar_expect_tx(&bar[sl], 32768);
        // box = [run 16 amps][1][64 rows]; quarter q = rows 64 q .. 64 q + 63 (dim 3)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
            "[%6];" ::"r"(smem_u32(slots + (size_t)sl * 2048)),
            "l"((uint64_t)&in), "r"(0), "r"((int)T), "r"(0), "r"(q), "r"(smem_u32(&bar[sl]))
            : "memory");
    };
    if (threadIdx.x == 0)
        for (uint64_t s = 0; s < 7; ++s) issue(s);
    for (uint64_t j = 0;; ++j) {
        const uint64_t T = blockIdx.x + j * gridDim.x;
        if (T >= ntiles) break;
        const uint32_t s0 = (uint32_t)((4 * j) % 7);
        for (int q = 0; q < 4; ++q) mbar_wait(&bar[(4 * j + q) % 7], (uint32_t)(((4 * j + q) / 7) & 1));
        double2 v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t e = threadIdx.x + 256 * k;
            uint32_t sl = s0 + (e >> 11);
            if (sl >= 7) sl -= 7;
            v[k] = slots[sl * 2048 + (e & 2047)];
        }
        if (MODE == 0) {
            __syncthreads();
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint32_t e = (threadIdx.x * 32 + k) ^ ((threadIdx.x) & 7);
                uint32_t sl = s0 + (e >> 11);
                if (sl >= 7) sl -= 7;
                slots[sl * 2048 + (e & 2047)] = v[k];
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint32_t e = (threadIdx.x * 32 + k) ^ ((threadIdx.x) & 7);
                uint32_t sl = s0 + (e >> 11);
                if (sl >= 7) sl -= 7;
                v[k] = slots[sl * 2048 + (e & 2047)];
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0)
            for (uint64_t s = 4 * j + 7; s < 4 * j + 11; ++s) issue(s);
#pragma unroll
        for (int k = 0; k < 32; ++k)
            __stcs(out + T * 8192 + threadIdx.x + 256 * k, make_double2(v[k].x + 1.0, v[k].y));
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv)
{
    const uint64_t n = 1ull << N;
    double2 *x, *y;
    cudaMalloc(&x, n * 16);
    cudaMalloc(&y, n * 16);
    cudaMemset(x, 0, n * 16);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)p;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t smem = 3 * TILE_BYTES + 64;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint64_t ntiles = n >> TB;
    for (int r = 1; r <= 6; ++r) {
        const int mid = N - TB;
        CUtensorMap m;
        if (TB - r > 8) continue;   // rows > 256: see k_q13 for the 4-D form
        cuuint64_t gdim[3] = {(cuuint64_t)2 << r, (cuuint64_t)1 << mid, (cuuint64_t)1 << (TB - r)};
        cuuint64_t gstr[2] = {(cuuint64_t)16 << r, (cuuint64_t)16 << (r + mid)};
        cuuint32_t box[3] = {2u << r, 1u, 1u << (TB - r)};
        cuuint32_t es[3] = {1, 1, 1};
        for (int prom = 0; prom < 2; ++prom) {
            CUresult cr = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE,
                              prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) {
                printf("encode failed r=%d: %d\n", r, (int)cr);
                continue;
            }
            k_tma<<<sms, 256, smem>>>(m, y, r, ntiles);
            cudaEventRecord(e0);
            for (int rep = 0; rep < 5; ++rep) k_tma<<<sms, 256, smem>>>(m, y, r, ntiles);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"kind\": \"tma\", \"run_bytes\": %d, \"prom256\": %d, \"tbs\": %.3f, \"err\": \"%s\"}\n", 16 << r, prom,
                   5.0 * n * 32 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
        for (int per = 1; per <= 2; ++per) {
            k_ldg<<<sms * per, 256>>>(x, y, r, ntiles);
            cudaEventRecord(e0);
            for (int rep = 0; rep < 5; ++rep) k_ldg<<<sms * per, 256>>>(x, y, r, ntiles);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"kind\": \"ldg\", \"run_bytes\": %d, \"ctas_per_sm\": %d, \"tbs\": %.3f, \"err\": \"%s\"}\n", 16 << r,
                   per, 5.0 * n * 32 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
    }
    // 13-bit tiles: run 16 amps (256 B) x 512 rows (top 9 positions), quarter = 128 rows
    {
        const int r = 4, rows = 9, mid = N - 13;
        CUtensorMap m;
        cuuint64_t gdim[4] = {(cuuint64_t)2 << r, (cuuint64_t)1 << mid, (cuuint64_t)128, (cuuint64_t)4};
        cuuint64_t gstr[3] = {(cuuint64_t)16 << r, (cuuint64_t)16 << (r + mid), (cuuint64_t)16 << (r + mid + 7)};
        cuuint32_t box[4] = {2u << r, 1u, 128u, 1u};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult cr = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        (void)rows;
        const size_t sm13 = 7 * 32768 + 64;
        cudaFuncSetAttribute(k_q13<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm13);
        cudaFuncSetAttribute(k_q13<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm13);
        const uint64_t nt13 = n >> 13;
        for (int mode = 0; mode < 2; ++mode) {
            if (cr != CUDA_SUCCESS) { printf("encode13 failed %d\n", (int)cr); break; }
            auto go = [&]() { if (mode) k_q13<1><<<sms, 256, sm13>>>(m, y, nt13); else k_q13<0><<<sms, 256, sm13>>>(m, y, nt13); };
            go();
            cudaEventRecord(e0);
            for (int rep = 0; rep < 5; ++rep) go();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"kind\": \"q13\", \"mode\": %d, \"run_bytes\": 256, \"tbs\": %.3f, \"err\": \"%s\"}\n", mode,
                   5.0 * n * 32 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
