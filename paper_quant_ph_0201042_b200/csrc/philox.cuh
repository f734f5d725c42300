// philox.cuh -- the library's counter-based RNG (reading R1).
//
// Philox4x32-10 (Salmon et al., SC'11) usable from host and device code.
// This is the GPU path's own implementation; the oracle has an independent
// one (oracle/oracle.c).  Both are pinned to the published known answers.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define QS_HD __host__ __device__ __forceinline__
#else
#define QS_HD inline
#endif

namespace qs {

struct u64x2 { uint64_t a, b; };

QS_HD void mulhilo32(uint32_t m, uint32_t x, uint32_t &hi, uint32_t &lo)
{
#ifdef __CUDA_ARCH__
    hi = __umulhi(m, x);
    lo = m * x;
#else
    uint64_t p = (uint64_t)m * (uint64_t)x;
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
#endif
}

// Ten Philox4x32 rounds on counter (c0..c3) with key (k0, k1).
QS_HD void philox10(uint32_t &c0, uint32_t &c1, uint32_t &c2, uint32_t &c3,
                    uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hA, lA, hB, lB;
        mulhilo32(0xD2511F53u, c0, hA, lA);
        mulhilo32(0xCD9E8D57u, c2, hB, lB);
        const uint32_t t0 = hB ^ c1 ^ k0, t2 = hA ^ c3 ^ k1;
        c0 = t0; c1 = lB; c2 = t2; c3 = lA;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// draw(seed, tag, i, j): key = seed, counter = (i, j, tag).
QS_HD u64x2 draw(uint64_t seed, uint32_t tag, uint64_t i, uint32_t j)
{
    uint32_t c0 = (uint32_t)i, c1 = (uint32_t)(i >> 32), c2 = j, c3 = tag;
    philox10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
    u64x2 r;
    r.a = (uint64_t)c0 | ((uint64_t)c1 << 32);
    r.b = (uint64_t)c2 | ((uint64_t)c3 << 32);
    return r;
}

QS_HD double u01(uint64_t a) { return (double)(a >> 11) * (1.0 / 9007199254740992.0); }
QS_HD double u01o(uint64_t a) { return (double)((a >> 11) + 1) * (1.0 / 9007199254740992.0); }

QS_HD uint64_t uint_below(uint64_t a, uint64_t m)
{
#ifdef __CUDA_ARCH__
    return __umul64hi(a, m);
#else
    return (uint64_t)(((unsigned __int128)a * m) >> 64);
#endif
}

}  // namespace qs
