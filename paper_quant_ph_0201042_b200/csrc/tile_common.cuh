// tile_common.cuh -- device helpers shared by the fused tile kernels
// (k_tile.cu: register/L2 path, k_tma.cu: TMA-pipelined path).
#pragma once
#include "qsim_internal.h"

namespace qs {
namespace tile {

constexpr int NS = 1 << kRegBits;   // slots per thread

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// 16-byte-granular XOR swizzle inside the tile (avoids bank conflicts when a
// quarter-warp walks tile bits >= 3).
__device__ __forceinline__ uint32_t swz(uint32_t ti)
{
    uint32_t f = (ti >> 3) ^ (ti >> 6) ^ (ti >> 9) ^ (ti >> 12);
    return ti ^ (f & 7u);
}

__device__ __forceinline__ uint32_t thread_part(const TileMap &m, int nthr_bits, uint32_t tid)
{
    uint32_t ti = 0;
    for (int t = 0; t < nthr_bits; ++t) ti |= ((tid >> t) & 1u) << m.order[t];
    return ti;
}

// exp(+-2 pi i t / 2^W) from the root table (tab[k] = exp(+-2 pi i k/1024))
// and a Taylor series for the remainder angle (|theta| < 2 pi / 1024).
// tw = +-2 pi / 2^W (sign = direction of the transform).
__device__ __forceinline__ double2 root_of_unity(uint64_t t, int W, const double2 *tab, double tw)
{
    if (W <= 10) return tab[(uint32_t)(t << (10 - W)) & 1023u];
    const uint64_t hi = t >> (W - 10);
    const uint64_t lo = t & ((1ull << (W - 10)) - 1);
    double2 p = tab[(uint32_t)hi & 1023u];
    if (lo) {
        const double th = (double)lo * tw;
        const double t2 = th * th;
        const double c = fma(fma(fma(-t2, 1.0 / 720.0, 1.0 / 24.0), t2, -0.5), t2, 1.0);
        const double s = th * fma(fma(fma(-t2, 1.0 / 5040.0, 1.0 / 120.0), t2, -1.0 / 6.0), t2, 1.0);
        p = cmul(p, make_double2(c, s));
    }
    return p;
}

// compile-time-direction rotation c * exp(+-i pi / 2^d), d = 1, 2, 3
template <bool INV>
__device__ __forceinline__ double2 rot_c(double2 c, int d)
{
    if (d == 1) return INV ? make_double2(c.y, -c.x) : make_double2(-c.y, c.x);
    if (d == 2) {
        const double r = 0.70710678118654752440;
        return INV ? make_double2((c.x + c.y) * r, (c.y - c.x) * r) : make_double2((c.x - c.y) * r, (c.y + c.x) * r);
    }
    return cmul(c, make_double2(0.92387953251128675613, INV ? -0.38268343236508977173 : 0.38268343236508977173));
}

__device__ __forceinline__ void tile_store(double2 *buf, uint32_t i, double2 v) { buf[i] = v; }
__device__ __forceinline__ double2 tile_load(const double2 *buf, uint32_t i) { return buf[i]; }

// c * exp(+-i pi / 2^d) for d = 1, 2, 3 (sg = +-1: direction of the transform)
__device__ __forceinline__ double2 rot(double2 c, int d, double sg)
{
    if (d == 1) return make_double2(-sg * c.y, sg * c.x);
    if (d == 2) {
        const double r = 0.70710678118654752440;
        return make_double2((c.x - sg * c.y) * r, (c.y + sg * c.x) * r);
    }
    return cmul(c, make_double2(0.92387953251128675613, sg * 0.38268343236508977173));
}


// Barrier among the threads that own the tile: the whole CTA (register
// path) or the 256 compute threads of a warp-specialised CTA (named barrier 1).
template <bool NAMED>
__device__ __forceinline__ void tile_sync()
{
    if (NAMED) asm volatile("bar.sync 1, 256;" ::: "memory");
    else __syncthreads();
}

// The arithmetic of one QFT / H block on a tile held as 16 amplitudes per
// thread in map-0 order: twiddle of the earlier blocks' R_d gates (+ the
// 2^(-a/2) normalisation), then for every register map: transpose through
// the tile buffer (XOR-swizzled), per active wire the R_d phases of the
// earlier wires of this block and the unnormalised H.
template <int NM, bool NAMED>
__device__ __forceinline__ void tile_body(double2 (&v)[NS], const TilePass &tp, const uint32_t (&tpart)[NM],
                                          const uint32_t (&stp)[NM], const double2 *tab, double2 *tile,
                                          uint64_t T, uint64_t yt, uint32_t Jt, bool twid, uint32_t amask,
                                          double sg)
{
    // ---- twiddle of the earlier blocks' R_d gates + normalisation
    if (twid) {
        uint64_t Y = tp.y_const + yt;
        for (int e = 0; e < tp.n_ef; ++e) Y += ((T >> tp.ef_bit[e]) & 1u) << tp.ef_w[e];
        if (tp.twiddle_fast) {
            // J = Jt + sum_b k_b jwin[b]  ->  phase(k) = A * prod_b beta_b^{k_b},
            // applied progressively (no table of 16 phases in registers)
            const double2 A = root_of_unity(Y * Jt, tp.W, tab, tp.tw);
            const double2 As = make_double2(A.x * tp.scale, A.y * tp.scale);
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = cmul(v[k], As);
#pragma unroll
            for (int b = 0; b < kRegBits; ++b) {
                if (!tp.jwin[b]) continue;
                const double2 beta = root_of_unity(Y * tp.jwin[b], tp.W, tab, tp.tw);
#pragma unroll
                for (int k = 0; k < NS; ++k)
                    if (k & (1 << b)) v[k] = cmul(v[k], beta);
            }
        } else {
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                uint32_t ti = tpart[0];
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
                    if (k & (1 << b)) ti |= 1u << tp.map[0].win[b];
                uint64_t Yk = Y - yt;
                for (int e = 0; e < tp.n_et; ++e) Yk += (uint64_t)((ti >> tp.et_bit[e]) & 1u) << tp.et_w[e];
                const uint32_t J = __brev(ti & amask) >> (32 - tp.a);
                const double2 r = root_of_unity(Yk * J, tp.W, tab, tp.tw);
                v[k] = cmul(v[k], make_double2(r.x * tp.scale, r.y * tp.scale));
            }
        }
    } else if (tp.scale != 1.0) {
#pragma unroll
        for (int k = 0; k < NS; ++k) v[k] = make_double2(v[k].x * tp.scale, v[k].y * tp.scale);
    }
    // ---- register maps
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        if (m > 0) {
            uint32_t s[NS];
            s[0] = stp[m - 1];
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int j = 0; j < (1 << b); ++j) s[j | (1 << b)] = s[j] ^ tp.wswz[m - 1][b];
            tile_sync<NAMED>();   // previous readers of the tile buffer are done
#pragma unroll
            for (int k = 0; k < NS; ++k) tile[s[k]] = v[k];
            s[0] = stp[m];
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int j = 0; j < (1 << b); ++j) s[j | (1 << b)] = s[j] ^ tp.wswz[m][b];
            tile_sync<NAMED>();
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = tile[s[k]];
        }
        const TileMap &mp = tp.map[m];
        if (mp.ucnt > 0) {
            const int w0 = mp.win[0];   // compute windows are contiguous: win[b] = w0 + b
#pragma unroll
            for (int rb = 0; rb < kRegBits; ++rb) {
                const int u = w0 + rb;
                if (u < mp.ustart || u >= mp.ustart + mp.ucnt) continue;
                if (!tp.hadamard_only && u > 0) {
                    // exp(i pi sum_{u'<u} y_u' 2^(u'-u)) on b_u = 1: thread part
                    // from the root table, window part = products of R_1..R_3
                    const double2 P = tab[((tpart[m] & ((1u << u) - 1u)) << (9 - u)) & 1023u];
#pragma unroll
                    for (int k = 0; k < NS; ++k) {
                        if (!(k & (1 << rb))) continue;
                        double2 x = cmul(v[k], P);
#pragma unroll
                        for (int r2 = 0; r2 < rb; ++r2)
                            if (k & (1 << r2)) x = rot(x, rb - r2, sg);
                        v[k] = x;
                    }
                }
                // H (unnormalised): (x, y) -> (x + y, x - y)
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    if (k & (1 << rb)) continue;
                    const double2 x = v[k], y = v[k | (1 << rb)];
                    v[k] = make_double2(x.x + y.x, x.y + y.y);
                    v[k | (1 << rb)] = make_double2(x.x - y.x, x.y - y.y);
                }
            }
        }
    }
}

}  // namespace tile
}  // namespace qs
