// k_grover.cu -- Grover iterations (§5.3), fused.
//
// One G-iteration is -H_n V_{f0} H_n V_{fk}.  Since -H_n V_{f0} H_n =
// 2|s><s| - I, the iteration is alpha_k <- -alpha_k followed by
// alpha <- 2 mean(alpha) - alpha (R17; the oracle applies the
// literal H_n / V_f0 / H_n sequence and the tests compare the two).
// Each iteration is ONE kernel over the state: every block updates a
// contiguous chunk and accumulates the sum of its new amplitudes; the last
// block to finish (atomic ticket) adds the block partials in a fixed tree
// order, forms the mean needed by the next iteration, (S - 2 alpha_k) / N,
// and records |alpha_k|^2 for this iteration.  At n = 20 the 16 MiB state
// stays resident in the 126 MB L2, so an iteration costs one L2 read+write
// of the state plus one launch.
#include <cooperative_groups.h>
#include <cstdlib>

#include "qsim_internal.h"

namespace qs {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 1024;

struct GroverCtl {
    double2 mean;
    unsigned int ticket;
    unsigned int pad;
    double2 part[kMaxBlocks];
};

__device__ __forceinline__ double2 warp_sum2(double2 v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

__device__ double2 block_sum2(double2 v, double2 *sh)
{
    v = warp_sum2(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double2 t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : make_double2(0.0, 0.0);
    if (w == 0) t = warp_sum2(t);
    if (threadIdx.x == 0) sh[0] = t;
    __syncthreads();
    return sh[0];
}

// init != 0: only sum the current state and form the first mean.
__global__ void __launch_bounds__(kThreads) k_grover_iter(double2 *__restrict__ psi, uint64_t N,
                                                          uint64_t chunk, uint64_t k,
                                                          GroverCtl *__restrict__ ctl,
                                                          double *__restrict__ trace, int t, int init)
{
    __shared__ double2 sh[32];
    __shared__ int s_last;
    const double2 mean = ctl->mean;
    const double m2x = 2.0 * mean.x, m2y = 2.0 * mean.y;
    const uint64_t b0 = (uint64_t)blockIdx.x * chunk;
    const uint64_t b1 = b0 + chunk < N ? b0 + chunk : N;
    double2 acc = make_double2(0.0, 0.0);
    for (uint64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
        double2 a = psi[i];
        if (!init) {
            if (i == k) { a.x = -a.x; a.y = -a.y; }        // V_{f_k}
            a = make_double2(m2x - a.x, m2y - a.y);        // 2|s><s| - I
            psi[i] = a;
        }
        acc.x += a.x;
        acc.y += a.y;
    }
    const double2 s = block_sum2(acc, sh);
    if (threadIdx.x == 0) {
        ctl->part[blockIdx.x] = s;
        __threadfence();
        const unsigned tk = atomicAdd(&ctl->ticket, 1u);
        s_last = tk == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // fixed-order tree over the block partials
    double2 v = make_double2(0.0, 0.0);
    for (unsigned j = threadIdx.x; j < gridDim.x; j += blockDim.x) {
        const double2 pj = __ldcg(&ctl->part[j]);
        v.x += pj.x;
        v.y += pj.y;
    }
    const double2 S = block_sum2(v, sh);
    if (threadIdx.x == 0) {
        const double2 ak = __ldcg(&psi[k]);
        const double inv = 1.0 / (double)N;
        ctl->mean = make_double2((S.x - 2.0 * ak.x) * inv, (S.y - 2.0 * ak.y) * inv);
        if (!init && trace) trace[t] = fma(ak.x, ak.x, ak.y * ak.y);
        ctl->ticket = 0;
        __threadfence();
    }
}

// Persistent variant for states that fit in shared memory across the GPU
// (n <= 20: 2^20 amplitudes = 128 CTAs x 8192 x 16 B): one cooperative
// launch runs every iteration; each CTA keeps its contiguous chunk of the
// state in shared memory for the whole search, so an iteration costs no
// DRAM/L2 traffic for the state -- only the block partial sums
// (double-buffered by iteration parity) and one grid barrier.  Every block
// reduces the partials in the same fixed order, so all blocks compute the
// identical mean.
namespace cg = cooperative_groups;

constexpr int kPersistThreads = 512;
constexpr int kRegsThreads = 256;
#ifndef GROVER_BACKOFF_NS
#define GROVER_BACKOFF_NS 32
#endif   // k_grover_regs: fewer, fatter threads (cheaper CTA barriers / trees)

__global__ void __launch_bounds__(kPersistThreads) k_grover_persist(double2 *__restrict__ psi, uint64_t N, uint64_t chunk,
                                                                    uint64_t k, int iters, double *__restrict__ trace,
                                                                    double2 *__restrict__ part, double2 *__restrict__ akbuf)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double2 st[];
    __shared__ double2 sh[32];
    __shared__ double2 s_mean;
    const unsigned nb = gridDim.x;
    const uint64_t base = (uint64_t)blockIdx.x * chunk;
    const bool own_k = k >= base && k < base + chunk;
    const uint32_t kl = (uint32_t)(k - base);
    double2 acc = make_double2(0.0, 0.0);
    for (uint32_t i = threadIdx.x; i < chunk; i += blockDim.x) {
        const double2 a = psi[base + i];
        st[i] = a;
        acc.x += a.x;
        acc.y += a.y;
    }
    auto publish = [&](int p, double2 a) {
        const double2 s = block_sum2(a, sh);
        if (threadIdx.x == 0) part[(size_t)p * nb + blockIdx.x] = s;
        grid.sync();
        if (threadIdx.x < 32) {
            double2 t = make_double2(0.0, 0.0);
            for (unsigned b = threadIdx.x; b < nb; b += 32) {
                const double2 q = __ldcg(&part[(size_t)p * nb + b]);
                t.x += q.x;
                t.y += q.y;
            }
            t = warp_sum2(t);
            if (threadIdx.x == 0) {
                const double2 ak = __ldcg(&akbuf[p]);
                const double inv = 1.0 / (double)N;
                s_mean = make_double2((t.x - 2.0 * ak.x) * inv, (t.y - 2.0 * ak.y) * inv);
            }
        }
        __syncthreads();
    };
    __syncthreads();
    if (own_k && threadIdx.x == 0) akbuf[0] = st[kl];
    publish(0, acc);
    for (int t = 0; t < iters; ++t) {
        const int p = (t + 1) & 1;
        const double2 mean = s_mean;
        const double m2x = 2.0 * mean.x, m2y = 2.0 * mean.y;
        acc = make_double2(0.0, 0.0);
        for (uint32_t i = threadIdx.x; i < chunk; i += blockDim.x) {
            double2 a = st[i];
            if (own_k && i == kl) { a.x = -a.x; a.y = -a.y; }   // V_{f_k}
            a = make_double2(m2x - a.x, m2y - a.y);             // 2|s><s| - I
            st[i] = a;
            acc.x += a.x;
            acc.y += a.y;
        }
        __syncthreads();
        if (own_k && threadIdx.x == 0) {
            const double2 ak = st[kl];
            akbuf[p] = ak;
            if (trace) trace[t] = fma(ak.x, ak.x, ak.y * ak.y);
        }
        publish(p, acc);
    }
    for (uint32_t i = threadIdx.x; i < chunk; i += blockDim.x) psi[base + i] = st[i];
}

// Register-resident variant (the default when the state fits): the 2^n
// amplitudes live in the registers of a co-resident grid (<= 16 per thread),
// and the per-iteration all-reduce is a slot exchange: every CTA publishes
// {sum of its amplitudes, alpha_k if it owns k} into its slot of a parity
// double buffer, arrives on a monotonic counter (red.release), one thread per
// CTA polls the counter (ld.acquire), then every CTA reads all slots and sums
// them in the same fixed order, so all CTAs form the identical mean.  Parity
// buffers make a slot safe to overwrite: a CTA can only publish iteration
// t+2 after every CTA has published t+1, i.e. finished reading t.  (Measured
// alternative: slots in NCCL's "LL" layout -- 64-bit words of {32 data bits,
// tag}, read by 128 pollers per CTA without the counter -- 2.7x slower.)
// CARRY: the amplitude sum is carried instead of re-reduced every
// iteration.  D = 2|s><s| - I has |s> as an eigenvector and is symmetric, so
// <s|D phi> = <s|phi> for every phi: the sum after an iteration is the sum
// after the phase flip, S - 2 alpha_k, and alpha_k itself becomes
// 2 (S - 2 alpha_k)/N + alpha_k.  Every CTA evolves (S, alpha_k) with exactly
// the floating-point operations the owner of alpha_k applies to its register,
// so all CTAs agree bit for bit with the state and no grid-wide exchange is
// needed after the first sum; every amplitude is still updated in every
// iteration.
template <int A, bool CARRY>
__global__ void __launch_bounds__(kRegsThreads, A <= 8 ? 2 : 1) k_grover_regs(double2 *__restrict__ psi, uint64_t N, uint64_t k,
                                                                   int iters, double *__restrict__ trace,
                                                                   double4 *__restrict__ slots,
                                                                   unsigned *__restrict__ tags)
{
    __shared__ double2 sh[32];
    __shared__ double4 s_tot;
    const unsigned nb = gridDim.x;
    const uint64_t chunk = (uint64_t)A * blockDim.x;
    const uint64_t base = (uint64_t)blockIdx.x * chunk;
    // slots of this thread inside the state (all A but in the last CTA)
    const uint64_t first = base + threadIdx.x;
    const uint64_t nv_all = first >= N ? 0 : (N - first + blockDim.x - 1) / blockDim.x;
    const int nv = nv_all > (uint64_t)A ? A : (int)nv_all;
    double2 v[A];
#pragma unroll
    for (int j = 0; j < A; ++j)   // ragged last CTA: slots past N hold 0, evolve harmlessly, are never stored
        v[j] = j < nv ? psi[base + threadIdx.x + (uint64_t)j * blockDim.x] : make_double2(0.0, 0.0);
    // the owner of k: thread / register slot (static index via the unrolled loops)
    const bool own_k = k >= base && k < base + chunk;
    const uint32_t kl = (uint32_t)(k - base);
    const bool own_t = own_k && (kl % blockDim.x) == threadIdx.x;
    const int kj = (int)(kl / blockDim.x);
    const double inv = 1.0 / (double)N;

    auto exchange = [&](int it) {   // publish the partial of iteration `it` (-1: initial state), gather the total
        double2 acc = make_double2(0.0, 0.0), ak = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < A; ++j) {
            if (j >= nv) break;   // ragged: slots past N are not amplitudes
            acc.x += v[j].x;
            acc.y += v[j].y;
            if (own_t && j == kj) ak = v[j];
        }
        acc = warp_sum2(acc);
        ak = warp_sum2(ak);
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        __shared__ double2 sak[32];
        if (l == 0) {
            sh[w] = acc;
            sak[w] = ak;
        }
        __syncthreads();
        if (w == 0) {
            // warp 0 does the rest: CTA partial (fixed shuffle tree), publish,
            // arrive on the counter and wait, then gather every CTA's slot
            // (lane l: slots l, l+32, ... in that order, then the fixed xor
            // tree) -- one CTA barrier per exchange besides the partials'
            const unsigned p = (unsigned)(it + 1) & 1u;
            const int nw = (int)(blockDim.x >> 5);
            double2 t = l < nw ? sh[l] : make_double2(0.0, 0.0);
            double2 a = l < nw ? sak[l] : make_double2(0.0, 0.0);
            t = warp_sum2(t);
            a = warp_sum2(a);
            if (l == 0) {
                slots[(size_t)p * nb + blockIdx.x] = make_double4(t.x, t.y, a.x, a.y);
                // monotonic counter compared wrap-safe: it wraps after ~2^32 / nb
                // iterations, but no CTA runs more than one exchange ahead
                const unsigned target = nb * (unsigned)(it + 2);
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(tags) : "memory");
                unsigned got;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(tags) : "memory");
                while ((int)(got - target) < 0) {
                    __nanosleep(GROVER_BACKOFF_NS);
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(tags) : "memory");
                }
            }
            __syncwarp();
            double4 q = make_double4(0.0, 0.0, 0.0, 0.0);
            for (unsigned b = l; b < nb; b += 32) {
                const double2 *sp = reinterpret_cast<const double2 *>(slots + (size_t)p * nb + b);
                const double2 q0 = __ldcg(sp), q1 = __ldcg(sp + 1);
                q.x += q0.x;
                q.y += q0.y;
                q.z += q1.x;
                q.w += q1.y;
            }
            const double2 s1 = warp_sum2(make_double2(q.x, q.y));
            const double2 s2 = warp_sum2(make_double2(q.z, q.w));
            if (l == 0) s_tot = make_double4(s1.x, s1.y, s2.x, s2.y);
        }
        __syncthreads();
    };

    exchange(-1);
    double4 cur = s_tot;   // (S, alpha_k) -- carried in registers when CARRY
    for (int t = 0; t < iters; ++t) {
        const double4 T = CARRY ? cur : s_tot;   // sum S and alpha_k of the previous iteration
        // after V_{f_k} the sum is S - 2 alpha_k; 2|s><s| - I maps a -> 2 mean - a
        const double sfx = T.x - 2.0 * T.z, sfy = T.y - 2.0 * T.w;
        const double m2x = 2.0 * sfx * inv, m2y = 2.0 * sfy * inv;
        if (CARRY) {
            // alpha_k lives in cur (bit-identical in every CTA), so the
            // owner's register slot is left to the plain update and replaced
            // by cur at the store: no per-amplitude sign select, 2 DADD per
            // amplitude
#pragma unroll
            for (int j = 0; j < A; ++j) v[j] = make_double2(m2x - v[j].x, m2y - v[j].y);
        } else {
#pragma unroll
            for (int j = 0; j < A; ++j) {
                double2 a = v[j];
                if (own_t && j == kj) { a.x = -a.x; a.y = -a.y; }   // V_{f_k}
                v[j] = make_double2(m2x - a.x, m2y - a.y);
            }
        }
        if (CARRY) {
            // the owner's update of alpha_k, m2 - (-alpha_k), with the same operations
            cur = make_double4(sfx, sfy, m2x - (-T.z), m2y - (-T.w));
            if (blockIdx.x == 0 && threadIdx.x == 0 && trace) trace[t] = fma(cur.z, cur.z, cur.w * cur.w);
        } else {
            exchange(t);
            if (blockIdx.x == 0 && threadIdx.x == 0 && trace) trace[t] = fma(s_tot.z, s_tot.z, s_tot.w * s_tot.w);
        }
    }
#pragma unroll
    for (int j = 0; j < A; ++j)
        if (j < nv)
            psi[base + threadIdx.x + (uint64_t)j * blockDim.x] =
                CARRY && iters > 0 && own_t && j == kj ? make_double2(cur.z, cur.w) : v[j];
}

}  // namespace

static bool try_persist(Handle *h, uint64_t mark, int iters, double *d_trace)
{
    const uint64_t N = h->local_dim();
    // the largest power-of-two grid that is co-resident (one CTA per SM)
    uint64_t blocks = 1;
    while (blocks * 2 <= (uint64_t)h->num_sms && blocks * 2 <= N / kPersistThreads) blocks *= 2;
    const uint64_t chunk = N / blocks;
    const size_t smem = chunk * sizeof(double2);
    if (smem > 200 * 1024 || blocks > kMaxBlocks) return false;
    cudaFuncSetAttribute(k_grover_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_grover_persist, kPersistThreads, smem);
    if (per_sm < 1 || blocks > (uint64_t)per_sm * h->num_sms) return false;
    ensure_red(h, 8 + 4 * (size_t)blocks + 8);
    double2 *part = reinterpret_cast<double2 *>(h->d_red + 8);
    double2 *akbuf = part + 2 * blocks;
    void *args[] = {(void *)&h->psi, (void *)&N,      (void *)&chunk, (void *)&mark,
                    (void *)&iters,  (void *)&d_trace, (void *)&part,  (void *)&akbuf};
    prof_begin(h);
    cudaError_t e = cudaLaunchCooperativeKernel((void *)k_grover_persist, dim3((unsigned)blocks), dim3(kPersistThreads),
                                                args, smem, h->stream);
    prof_end(h, "k_grover_persist", N * 32);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}

static bool try_regs(Handle *h, uint64_t mark, int iters, double *d_trace)
{
    const uint64_t N = h->local_dim();
    // QSIM_GROVER_REDUCE: re-reduce the sum every iteration (measurement / cross-check knob)
    static const bool reduce = getenv("QSIM_GROVER_REDUCE") != nullptr;
    // amplitudes per thread: the instantiated A >= per
    static const int kA[] = {1, 2, 4, 8, 12, 16, 20, 24, 28, 32};
    auto inst = [&](int A) -> void * {
        switch (A) {
        case 1: return reduce ? (void *)k_grover_regs<1, false> : (void *)k_grover_regs<1, true>;
        case 2: return reduce ? (void *)k_grover_regs<2, false> : (void *)k_grover_regs<2, true>;
        case 4: return reduce ? (void *)k_grover_regs<4, false> : (void *)k_grover_regs<4, true>;
        case 8: return reduce ? (void *)k_grover_regs<8, false> : (void *)k_grover_regs<8, true>;
        case 12: return reduce ? (void *)k_grover_regs<12, false> : (void *)k_grover_regs<12, true>;
        case 16: return reduce ? (void *)k_grover_regs<16, false> : (void *)k_grover_regs<16, true>;
        case 20: return reduce ? (void *)k_grover_regs<20, false> : (void *)k_grover_regs<20, true>;
        case 24: return reduce ? (void *)k_grover_regs<24, false> : (void *)k_grover_regs<24, true>;
        case 28: return reduce ? (void *)k_grover_regs<28, false> : (void *)k_grover_regs<28, true>;
        default: return reduce ? (void *)k_grover_regs<32, false> : (void *)k_grover_regs<32, true>;
        }
    };
    // one CTA per SM (every CTA co-resident: the first sum is a grid-wide
    // exchange), the state spread over all of them: the smallest instantiated
    // A with A x 256 x SMs >= N, the last CTA ragged (n = 20: A = 28 over 147
    // CTAs instead of 32 over 128 -- the FP64 update time per iteration is
    // set by the busiest SM)
    const uint64_t per_min = (N + (uint64_t)h->num_sms * kRegsThreads - 1) / ((uint64_t)h->num_sms * kRegsThreads);
    int A = 0;
    for (int a : kA)
        if ((uint64_t)a >= per_min) { A = a; break; }
    if (!A) return false;
    const uint64_t blocks = (N + (uint64_t)A * kRegsThreads - 1) / ((uint64_t)A * kRegsThreads);
    int per_sm = 0;
    void *fn = inst(A);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kRegsThreads, 0);
    if (per_sm < 1 || blocks > (uint64_t)per_sm * h->num_sms) return false;
    // slots: 2 x blocks double4 (parity double buffer); tags[0]: the arrival counter
    const size_t nd = 8 * blocks + blocks + 16;
    ensure_red(h, 8 + nd);
    double4 *slots = reinterpret_cast<double4 *>(h->d_red + 8);
    unsigned *tags = reinterpret_cast<unsigned *>(h->d_red + 8 + 8 * blocks);
    cudaMemsetAsync(tags, 0, 2 * blocks * sizeof(unsigned), h->stream);
    void *args[] = {(void *)&h->psi, (void *)&N, (void *)&mark, (void *)&iters, (void *)&d_trace, (void *)&slots,
                    (void *)&tags};
    prof_begin(h);
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)blocks), dim3(kRegsThreads), args, 0, h->stream);
    prof_end(h, "k_grover_regs", N * 32);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}

void launch_grover(Handle *h, uint64_t mark_local, int mark_rank, int iters, double *d_trace)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    (void)mark_rank;
    const uint64_t N = h->local_dim();
    if (!getenv("QSIM_NO_GROVER_REGS") && N >= 4096 && try_regs(h, mark_local, iters, d_trace)) return;
    // whole state in registers: <= 16 amplitudes per thread over the resident grid
    if (!getenv("QSIM_NO_GROVER_PERSIST") && N >= 4096 && try_persist(h, mark_local, iters, d_trace)) return;
    unsigned blocks = (unsigned)h->num_sms * 4;
    if (blocks > kMaxBlocks) blocks = kMaxBlocks;
    uint64_t chunk = (N + blocks - 1) / blocks;
    chunk = (chunk + kThreads - 1) / kThreads * kThreads;
    blocks = (unsigned)((N + chunk - 1) / chunk);
    const size_t need = (sizeof(GroverCtl) + sizeof(double) - 1) / sizeof(double);
    ensure_red(h, need + 8);
    GroverCtl *ctl = reinterpret_cast<GroverCtl *>(h->d_red + 8);
    cudaMemsetAsync(ctl, 0, sizeof(GroverCtl), h->stream);
    prof_begin(h);
    k_grover_iter<<<blocks, kThreads, 0, h->stream>>>(h->psi, N, chunk, mark_local, ctl, d_trace, 0, 1);
    prof_end(h, "k_grover_iter", N * 16);
    for (int t = 0; t < iters; ++t) {
        prof_begin(h);
        k_grover_iter<<<blocks, kThreads, 0, h->stream>>>(h->psi, N, chunk, mark_local, ctl, d_trace, t, 0);
        prof_end(h, "k_grover_iter", N * 32);
    }
}

}  // namespace qs
