// k_perm.cu -- basis permutations: modular multiplication / exponentiation
// applied as a permutation of amplitudes (§2.3.3; the
// paper's gate-level constant-adder circuit is replaced by its action, as in
// its own "semantic" Shor mode).  Integer work only; the
// result is bit-exact (amplitudes are moved, never recomputed).
//
// Fast path: the work register occupies the lowest wm local positions in
// value order (the canonical layout of configs[3]).  Then every run of 2^wm
// amplitudes shares one exponent value e, the permutation stays inside the
// run, and one CTA moves a run through shared memory in place: it computes
// c = base^e mod N (or the controlled multiplier) once, then gathers
// new[w'] = old[w' * c^-1 mod N] (w' < N; identity above, R10).
// HBM traffic = one read + one write of the state (32 B per amplitude).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "qsim_internal.h"
#include "mbar.cuh"

namespace qs {

namespace {

// x mod N for x < 2^64 with a precomputed floor((2^64-1)/N) (Barrett).
__device__ __forceinline__ uint64_t mod_barrett(uint64_t x, uint64_t N, uint64_t minv)
{
    uint64_t q = __umul64hi(x, minv);
    uint64_t r = x - q * N;
    while (r >= N) r -= N;
    return r;
}

__device__ uint64_t mulmod(uint64_t a, uint64_t b, uint64_t N, uint64_t minv)
{
    // a, b < N < 2^32 -> a*b < 2^64
    return mod_barrett(a * b, N, minv);
}

__device__ uint64_t powmod_dev(uint64_t base, uint64_t e, uint64_t N, uint64_t minv)
{
    uint64_t r = 1 % N, b = base % N;
    while (e) {
        if (e & 1) r = mulmod(r, b, N, minv);
        b = mulmod(b, b, N, minv);
        e >>= 1;
    }
    return r;
}

// inverse of c mod N (gcd(c, N) = 1), extended Euclid
__device__ uint64_t invmod_dev(uint64_t c, uint64_t N)
{
    int64_t t = 0, nt = 1;
    int64_t r = (int64_t)N, nr = (int64_t)(c % N);
    while (nr != 0) {
        const int64_t q = r / nr;
        int64_t tmp = t - q * nt; t = nt; nt = tmp;
        tmp = r - q * nr; r = nr; nr = tmp;
    }
    if (t < 0) t += (int64_t)N;
    return (uint64_t)t;
}

struct PermArgs {
    int kind;
    int wm;
    int em;
    int epos[40];          // exponent value bit b -> local position, or -1-g for rank bit g
    uint64_t cmask, cval;  // local control mask / values
    uint64_t ctrl_global_ok;
    uint64_t rank;         // this rank (global bits)
    uint64_t mult, base, N, minv;
    int wpos[40];          // generic path: work value bit b -> local position
    const uint32_t *table;
};

__device__ __forceinline__ uint64_t exponent_of(const PermArgs &a, uint64_t i)
{
    uint64_t e = 0;
    for (int b = 0; b < a.em; ++b) {
        const int p = a.epos[b];
        const uint64_t bit = p >= 0 ? (i >> p) & 1 : (a.rank >> (-1 - p)) & 1;
        e |= bit << b;
    }
    return e;
}

// one CTA per run of 2^wm amplitudes (work register = positions 0..wm-1)
__global__ void __launch_bounds__(256) k_perm_block(double2 *__restrict__ psi, uint64_t nruns,
                                                    PermArgs a)
{
    extern __shared__ double2 run[];
    __shared__ uint64_t s_cinv;
    __shared__ int s_active;
    const uint64_t len = 1ull << a.wm;
    for (uint64_t rix = blockIdx.x; rix < nruns; rix += gridDim.x) {
        double2 *g = psi + rix * len;
        const uint64_t base_i = rix * len;
        if (threadIdx.x == 0) {
            int active = a.ctrl_global_ok && ((base_i & a.cmask) == a.cval);
            uint64_t c = 1;
            if (active) {
                if (a.kind == QSIM_PERM_MODMUL) c = a.mult % a.N;
                else if (a.kind == QSIM_PERM_MODEXP) c = powmod_dev(a.base, exponent_of(a, base_i), a.N, a.minv);
            }
            if (a.kind != QSIM_PERM_TABLE && c == 1) active = 0;
            s_active = active;
            s_cinv = (active && a.kind != QSIM_PERM_TABLE) ? invmod_dev(c, a.N) : 1;
        }
        __syncthreads();
        if (s_active) {
            for (uint64_t w = threadIdx.x; w < len; w += blockDim.x) run[w] = g[w];
            __syncthreads();
            const uint64_t cinv = s_cinv;
            if (a.kind == QSIM_PERM_TABLE) {
                // new[table[v]] = old[v]
                for (uint64_t v = threadIdx.x; v < len; v += blockDim.x) g[a.table[v]] = run[v];
            } else {
                for (uint64_t w = threadIdx.x; w < len; w += blockDim.x) {
                    const uint64_t v = w < a.N ? mulmod(w, cinv, a.N, a.minv) : w;
                    g[w] = run[v];
                }
            }
        }
        __syncthreads();
    }
}

// Pipelined form of k_perm_block for MODMUL / MODEXP: persistent CTAs with a
// ring of kPermStages run buffers.  A producer warp (warp 8) forms each run's
// multiplier and issues its 1-D bulk copy as soon as the run's buffer is
// free (an "empty" mbarrier per stage, one arrival per consumer warp), so the
// HBM reads of later runs overlap the eight consumer warps' gather and
// store, and the consumers never wait on the producer's arithmetic.  The
// multiplier is a product of host tables, c = prod_{bit j of e} base^(2^j)
// and c^-1 = prod of their inverses (mod N): one lane per exponent bit and a
// shuffle-tree product, no serial powmod / extended Euclid per run.
constexpr int kPermStages = 4;
constexpr int kPermConsumers = 256;
struct PowTabs {
    uint64_t pw[40], inv[40];   // base^(2^j) mod N and its inverse; MODMUL: pw[0] = c, inv[0] = c^-1
};

__device__ __forceinline__ uint64_t warp_prod_mod(uint64_t x, uint64_t N, uint64_t minv)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = mulmod(x, __shfl_xor_sync(0xffffffffu, x, o), N, minv);
    return x;
}

__global__ void __launch_bounds__(kPermConsumers + 32) k_perm_ring(double2 *__restrict__ psi, uint64_t nruns,
                                                                   const __grid_constant__ PermArgs a,
                                                                   const __grid_constant__ PowTabs tb)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t len = 1u << a.wm;
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(bufs + (size_t)kPermStages * len);
    uint64_t *empty = full + kPermStages;
    __shared__ uint64_t s_cinv[kPermStages];
    __shared__ int s_act[kPermStages];
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    if (tid == 0) {
        for (int s = 0; s < kPermStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kPermConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid >= kPermConsumers) {
        // producer warp
        for (uint64_t k = 0;; ++k) {
            const uint64_t r = blockIdx.x + k * gridDim.x;
            if (r >= nruns) break;
            const int s = (int)(k % kPermStages);
            if (k >= (uint64_t)kPermStages) mbar_wait(&empty[s], (uint32_t)(((k / kPermStages) + 1) & 1));
            const uint64_t base_i = r << a.wm;
            int active = a.ctrl_global_ok && ((base_i & a.cmask) == a.cval);
            uint64_t c, ci;
            if (a.kind == QSIM_PERM_MODEXP) {
                const uint64_t e = exponent_of(a, base_i);
                const bool on = lane < (uint32_t)a.em && ((e >> lane) & 1u);
                c = warp_prod_mod(on ? tb.pw[lane] : 1, a.N, a.minv);
                ci = warp_prod_mod(on ? tb.inv[lane] : 1, a.N, a.minv);
            } else {
                c = tb.pw[0];
                ci = tb.inv[0];
            }
            if (c == 1 % a.N) active = 0;
            if (lane == 0) {
                s_act[s] = active;
                s_cinv[s] = ci;
                if (active) {
                    mbar_expect_tx(&full[s], len * 16u);
                    bulk_load_1d(bufs + (size_t)s * len, psi + base_i, len * 16u, &full[s]);
                } else {
                    mbar_arrive(&full[s]);
                }
            }
            __syncwarp();
        }
        return;
    }
    for (uint64_t k = 0;; ++k) {
        const uint64_t r = blockIdx.x + k * gridDim.x;
        if (r >= nruns) break;
        const int s = (int)(k % kPermStages);
        mbar_wait(&full[s], (uint32_t)((k / kPermStages) & 1));
        if (s_act[s]) {
            const uint64_t cinv = s_cinv[s];
            const double2 *run = bufs + (size_t)s * len;
            double2 *g = psi + (r << a.wm);
            for (uint32_t w = tid; w < len; w += kPermConsumers) {
                const uint64_t v = w < a.N ? mulmod(w, cinv, a.N, a.minv) : w;
                g[w] = run[v];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);   // this warp no longer reads stage s
    }
}

// generic out-of-place: dst[pi(i)] = src[i]
__global__ void __launch_bounds__(256) k_perm_generic(const double2 *__restrict__ src,
                                                      double2 *__restrict__ dst, uint64_t count,
                                                      PermArgs a)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        uint64_t v = 0;
        for (int b = 0; b < a.wm; ++b) v |= ((i >> a.wpos[b]) & 1) << b;
        uint64_t nv = v;
        if (a.ctrl_global_ok && (i & a.cmask) == a.cval) {
            if (a.kind == QSIM_PERM_TABLE) nv = a.table[v];
            else if (v < a.N) {
                uint64_t c = a.kind == QSIM_PERM_MODMUL ? a.mult % a.N
                                                        : powmod_dev(a.base, exponent_of(a, i), a.N, a.minv);
                nv = mulmod(v, c, a.N, a.minv);
            }
        }
        uint64_t j = i;
        for (int b = 0; b < a.wm; ++b) {
            const uint64_t m = 1ull << a.wpos[b];
            j = (j & ~m) | (((nv >> b) & 1) << a.wpos[b]);
        }
        dst[j] = src[i];
    }
}

}  // namespace

static uint64_t invmod_host(uint64_t c, uint64_t N)
{
    int64_t t = 0, nt = 1;
    int64_t r = (int64_t)N, nr = (int64_t)(c % N);
    while (nr != 0) {
        const int64_t q = r / nr;
        int64_t tmp = t - q * nt; t = nt; nt = tmp;
        tmp = r - q * nr; r = nr; nr = tmp;
    }
    if (t < 0) t += (int64_t)N;
    return (uint64_t)t % N;
}

int launch_perm(Handle *h, const PermDesc &d)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    PermArgs a;
    a.kind = d.kind;
    a.wm = d.wm;
    a.em = d.em;
    for (int b = 0; b < d.em; ++b) a.epos[b] = d.epos[b];
    for (int b = 0; b < d.wm; ++b) a.wpos[b] = d.wpos[b];
    a.cmask = d.cmask;
    a.cval = d.cval;
    a.ctrl_global_ok = 1;
    a.rank = d.rank_bits;
    a.mult = d.mult;
    a.base = d.base;
    a.N = d.modulus ? d.modulus : 1;
    a.minv = ~0ull / a.N;
    a.table = d.d_table;
    bool low_contig = true;
    for (int b = 0; b < d.wm; ++b) low_contig &= d.wpos[b] == b;
    // controls must not touch the work register in the block path
    low_contig &= (d.cmask & ((1ull << d.wm) - 1)) == 0;
    static const bool no_ring = getenv("QSIM_NO_PERM_RING") != nullptr;
    if (low_contig && d.wm >= 5 && d.wm <= 11 && d.em <= 32 && !no_ring &&
        (d.kind == QSIM_PERM_MODMUL || d.kind == QSIM_PERM_MODEXP)) {
        PowTabs tb;
        std::memset(&tb, 0, sizeof tb);
        if (d.kind == QSIM_PERM_MODEXP) {
            uint64_t p = a.base % a.N;
            for (int j = 0; j < d.em; ++j) {
                tb.pw[j] = p;
                tb.inv[j] = invmod_host(p, a.N);
                p = (uint64_t)((unsigned __int128)p * p % a.N);
            }
        } else {
            tb.pw[0] = a.mult % a.N;
            tb.inv[0] = invmod_host(tb.pw[0], a.N);
        }
        const uint64_t nruns = h->local_dim() >> d.wm;
        const size_t smem = ((size_t)kPermStages << d.wm) * sizeof(double2) + 2 * kPermStages * sizeof(uint64_t);
        static uint64_t attr = 0;
        if (first_use_on_device(attr))
            cudaFuncSetAttribute(k_perm_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_perm_ring, kPermConsumers + 32, smem);
        per_sm = std::max(1, std::min(per_sm, 3));
        const uint64_t cap = (uint64_t)h->num_sms * per_sm;
        prof_begin(h);
        k_perm_ring<<<(unsigned)(nruns < cap ? nruns : cap), kPermConsumers + 32, smem, h->stream>>>(h->psi, nruns,
                                                                                                   a, tb);
        prof_end(h, "k_perm_ring", h->local_dim() * 32);
    } else if (low_contig && d.wm <= 13 && d.wm >= 5) {
        const uint64_t nruns = h->local_dim() >> d.wm;
        const size_t smem = sizeof(double2) << d.wm;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_perm_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const uint64_t cap = (uint64_t)h->num_sms * (smem <= 32768 ? 6 : 1);
        prof_begin(h);
        k_perm_block<<<(unsigned)(nruns < cap ? nruns : cap), 256, smem, h->stream>>>(h->psi, nruns, a);
        prof_end(h, "k_perm_block", h->local_dim() * 32);
    } else {
        const uint64_t count = h->local_dim();
        if (int rc = ensure_scratch(h)) return rc;   // no room for the out-of-place permutation
        const uint64_t cap = (uint64_t)h->num_sms * 8;
        const uint64_t want = (count + 255) / 256;
        prof_begin(h);
        k_perm_generic<<<(unsigned)(want < cap ? want : cap), 256, 0, h->stream>>>(h->psi, h->scratch,
                                                                                 count, a);
        prof_end(h, "k_perm_generic", count * 32);
        swap_buffers(h);
    }
    return QSIM_OK;
}

}  // namespace qs
