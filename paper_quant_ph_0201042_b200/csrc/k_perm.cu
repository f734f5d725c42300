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
#include "qsim_internal.h"

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

void launch_perm(Handle *h, const PermDesc &d)
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
    if (low_contig && d.wm <= 13 && d.wm >= 5) {
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
        ensure_scratch(h);
        const uint64_t cap = (uint64_t)h->num_sms * 8;
        const uint64_t want = (count + 255) / 256;
        prof_begin(h);
        k_perm_generic<<<(unsigned)(want < cap ? want : cap), 256, 0, h->stream>>>(h->psi, h->scratch,
                                                                                 count, a);
        prof_end(h, "k_perm_generic", count * 32);
        swap_buffers(h);
    }
}

}  // namespace qs
