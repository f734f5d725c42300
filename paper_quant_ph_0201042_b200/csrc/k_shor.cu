// k_shor.cu -- Shor's factoring in the paper's semantic mode (SURVEY.md §8(f)
// row f3): the order-finding register prepared directly on the GPU, plus the
// classical post-processing on the host.
//
// Semantic mode: "the modular exponentiation are computed
// classically and the QFT is computed by the FFT algorithm ... the simulator
// does not need to generate the first register".  After step 3 of the
// algorithm and the measurement of f(a) = x^a mod N with
// outcome v, the exponent register holds the uniform superposition over
// {a : x^a = v (mod N)}.  k_shor_semantic evaluates that predicate for every
// basis index: each thread walks a strided run of exponents with one
// Montgomery (or Barrett) mulmod per amplitude (p <- p * x^32), so the write
// is coalesced and the kernel is bound by the 16 B/amplitude store, not by
// the arithmetic; the count pass that fixes the normalisation reads nothing.
//
// Post-processing (PAPER.md:851-859 steps 4-5; improvements 969-998) is
// host code: continued-fraction convergents of y / 2^m, the d+- gcd test,
// and the Prob_succ bound of PAPER.md:907-920.
#include "qsim_internal.h"
#include "../../include/qsim.h"

#include <cmath>

namespace qs {

namespace {

constexpr int kShorRun = 64;   // exponents per thread (lane-strided by 32)

// Modular products for N < 2^32.  Barrett: any N.  Montgomery (odd
// N < 2^31, the common case): values kept as a*2^32 mod N, one 32x32->64
// product, one 32-bit product and one 32x32->64 multiply-add per step.
struct Barrett {
    uint64_t N, minv;   // minv = floor((2^64 - 1) / N)
    __device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) const
    {
        const uint64_t t = a * b;                 // < 2^64 since a, b < N < 2^32
        uint64_t r = t - __umul64hi(t, minv) * N;
        while (r >= N) r -= N;
        return r;
    }
    __device__ __forceinline__ uint64_t one() const { return 1 % N; }
    __device__ __forceinline__ uint64_t from(uint64_t a) const { return a; }
};

struct Montgomery {
    uint32_t N, nprime;   // nprime = -N^-1 mod 2^32
    uint32_t r1;          // 2^32 mod N (the Montgomery form of 1)
    uint64_t r2;          // 2^64 mod N
    __device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) const
    {
        const uint64_t t = (uint64_t)(uint32_t)a * (uint32_t)b;
        const uint32_t m = (uint32_t)t * nprime;
        uint32_t u = (uint32_t)((t + (uint64_t)m * N) >> 32);   // < 2N; no overflow for N < 2^31
        if (u >= N) u -= N;
        return u;
    }
    __device__ __forceinline__ uint64_t one() const { return r1; }
    __device__ __forceinline__ uint64_t from(uint64_t a) const { return mul(a, r2); }
};

template <class Mod>
__device__ __forceinline__ uint64_t dev_powmod(const Mod &B, uint64_t xm, uint64_t e)
{
    uint64_t r = B.one(), b = xm;
    while (e) {
        if (e & 1) r = B.mul(r, b);
        b = B.mul(b, b);
        e >>= 1;
    }
    return r;
}

// Exponent a = a_base + local index; warp w of the grid owns 32*kShorRun
// consecutive local indices, lane l the ones = l (mod 32).  x, x32 and v
// arrive in the representation of Mod.
template <bool WRITE, class Mod>
__global__ void __launch_bounds__(256) k_shor_semantic(double2 *psi, uint64_t local_dim, uint64_t a_base,
                                                      Mod B, uint64_t x, uint64_t x32, uint64_t v,
                                                      double amp, unsigned long long *count)
{
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long c = 0;
    for (uint64_t w = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 32 * kShorRun < local_dim;
         w += warps) {
        const uint64_t i0 = w * 32 * kShorRun + lane;
        uint64_t p = dev_powmod(B, x, a_base + i0);
#pragma unroll 8
        for (int j = 0; j < kShorRun; ++j) {
            const uint64_t i = i0 + 32 * (uint64_t)j;
            if (i < local_dim) {   // shards below 2048 amplitudes
                const bool hit = p == v;
                if (WRITE)
                    __stcs(psi + i, make_double2(hit ? amp : 0.0, 0.0));
                else
                    c += hit;
            }
            p = B.mul(p, x32);
        }
    }
    if (!WRITE) {
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0 && c) atomicAdd(count, c);
    }
}

uint64_t host_powmod(uint64_t x, uint64_t e, uint64_t N)
{
    unsigned __int128 r = 1 % N, b = x % N;
    while (e) {
        if (e & 1) r = r * b % N;
        b = b * b % N;
        e >>= 1;
    }
    return (uint64_t)r;
}

uint64_t host_gcd(uint64_t a, uint64_t b)
{
    while (b) {
        const uint64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

}  // namespace

template <bool WRITE, class Mod>
static void launch_mod(Handle *h, unsigned grid, const Mod &B, uint64_t x, uint64_t x32, uint64_t v, double amp,
                       unsigned long long *d_count)
{
    k_shor_semantic<WRITE, Mod><<<grid, 256, 0, h->stream>>>(WRITE ? h->psi : nullptr, h->local_dim(),
                                                            (uint64_t)h->rank << h->nl, B, x, x32, v, amp, d_count);
}

static void launch_shor(Handle *h, bool write, uint64_t x, uint64_t N, uint64_t v, double amp,
                        unsigned long long *d_count)
{
    const uint64_t ld = h->local_dim();
    const uint64_t x32 = host_powmod(x, 32, N);
    const uint64_t warps_needed = (ld + 32 * kShorRun - 1) / (32 * kShorRun);
    const uint64_t blocks_needed = (warps_needed + 7) / 8;
    const uint64_t cap = (uint64_t)h->num_sms * 8;
    const unsigned grid = (unsigned)(blocks_needed < cap ? blocks_needed : cap);
    prof_begin(h);
    if ((N & 1) && N < (1ull << 31)) {
        Montgomery M;
        M.N = (uint32_t)N;
        uint32_t inv = 1;                       // Newton: N^-1 mod 2^32
        for (int k = 0; k < 5; ++k) inv *= 2u - (uint32_t)N * inv;
        M.nprime = 0u - inv;
        M.r1 = (uint32_t)((1ull << 32) % N);
        M.r2 = (uint64_t)(((unsigned __int128)1 << 64) % N);
        auto to = [&](uint64_t a) { return (uint64_t)(((unsigned __int128)a << 32) % N); };
        if (write) launch_mod<true>(h, grid, M, to(x), to(x32), to(v), amp, d_count);
        else launch_mod<false>(h, grid, M, to(x), to(x32), to(v), amp, d_count);
    } else {
        Barrett B{N, ~0ull / N};
        if (write) launch_mod<true>(h, grid, B, x, x32, v, amp, d_count);
        else launch_mod<false>(h, grid, B, x, x32, v, amp, d_count);
    }
    prof_end(h, write ? "k_shor_semantic_write" : "k_shor_semantic_count", write ? ld * 16 : 0);
}

void launch_shor_count(Handle *h, uint64_t x, uint64_t N, uint64_t v, unsigned long long *d_count)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    launch_shor(h, false, x, N, v, 0.0, d_count);
}

void launch_shor_write(Handle *h, uint64_t x, uint64_t N, uint64_t v, double amp)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    launch_shor(h, true, x, N, v, amp, nullptr);
}

}  // namespace qs

// ------------------------------------------------------------ host C-ABI part
using qs::host_gcd;
using qs::host_powmod;

extern "C" {

double qsim_shor_prob_succ(uint64_t n, uint64_t phi)
{
    if (n < 3 || phi == 0 || phi >= n) return NAN;
    const double euler_gamma = 0.577215664901532860606512090082;
    const double pi = 3.141592653589793238462643383280;
    const double p2 = 1.0 - (double)phi / (double)(n - 1);        // step 2 finds a factor
    const double p34 = 0.5 * (4.0 / (pi * pi)) * std::exp(-euler_gamma) / std::log(std::log((double)n));
    return p2 + (1.0 - p2) * p34;
}

int qsim_shor_candidates(uint64_t y, int m, uint64_t N, uint64_t *r_out, int cap)
{
    if (m < 1 || m > 62 || N < 2 || (!r_out && cap > 0) || cap < 0) return QSIM_EINVAL;
    const uint64_t M = 1ull << m;
    if (y == 0 || y >= M) return 0;
    // y/M = [c0; c1, c2, ...]; convergent h_k/k_k with h_k = c_k h_{k-1} + h_{k-2}
    uint64_t h2 = 0, h1 = 1, k2 = 1, k1 = 0;
    uint64_t a = y, b = M;
    int cnt = 0;
    while (b) {
        const uint64_t c = a / b, rem = a % b;
        a = b;
        b = rem;
        const uint64_t hk = c * h1 + h2, kk = c * k1 + k2;
        h2 = h1; h1 = hk;
        k2 = k1; k1 = kk;
        if (kk >= N) break;
        // accept when |y/M - hk/kk| <= 1/(2M), i.e. 2|y kk - hk M| <= kk
        const __int128 d = (__int128)y * kk - (__int128)hk * M;
        if (hk && 2 * (d < 0 ? -d : d) <= (__int128)kk) {
            if (cnt < cap) r_out[cnt] = kk;
            ++cnt;
        }
    }
    return cnt < cap ? cnt : cap;
}

uint64_t qsim_shor_try(uint64_t N, uint64_t x, uint64_t r, int gcd_check)
{
    if (N < 3 || r == 0 || (r & 1)) return 0;
    const bool period = host_powmod(x, r, N) == 1;
    if (!period && !gcd_check) return 0;
    const uint64_t z = host_powmod(x, r >> 1, N);
    if (!gcd_check && (z == 1 || z == N - 1)) return 0;
    for (const uint64_t t : {(z + N - 1) % N, (z + 1) % N}) {
        const uint64_t d = host_gcd(N, t);
        if (d > 1 && d < N) return d;
    }
    return 0;
}

}  // extern "C"
