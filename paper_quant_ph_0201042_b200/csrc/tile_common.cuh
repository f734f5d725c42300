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

__device__ __forceinline__ double2 cfma2(double2 u, double2 x, double2 v, double2 y)
{
    double re = fma(u.x, x.x, -u.y * x.y);
    double im = fma(u.x, x.y, u.y * x.x);
    re = fma(v.x, y.x, re);
    re = fma(-v.y, y.y, re);
    im = fma(v.x, y.y, im);
    im = fma(v.y, y.x, im);
    return make_double2(re, im);
}

// dense 2x2 on register bit RB for every slot pair whose window controls match
template <int RB, bool WC>
__device__ __forceinline__ void dense_rb(double2 (&v)[NS], const GOp &op)
{
    const double2 u0 = op.u[0], u1 = op.u[1], u2 = op.u[2], u3 = op.u[3];
    const uint32_t wm = op.wm, wv = op.wv;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if (k & (1 << RB)) continue;
        if (WC && ((k & wm) != wv)) continue;
        const double2 x = v[k], y = v[k | (1 << RB)];
        v[k] = cfma2(u0, x, u1, y);
        v[k | (1 << RB)] = cfma2(u2, x, u3, y);
    }
}

// diag(d0, d1) on window bit RB (D0ONE: d0 == 1, only the b = 1 half moves)
template <int RB, bool WC, bool D0ONE>
__device__ __forceinline__ void diag_rb(double2 (&v)[NS], const GOp &op)
{
    const double2 d0 = op.u[0], d1 = op.u[3];
    const uint32_t wm = op.wm, wv = op.wv;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if (WC && ((k & wm) != wv)) continue;
        if (k & (1 << RB)) v[k] = cmul(v[k], d1);
        else if (!D0ONE) v[k] = cmul(v[k], d0);
    }
}

// multiply every slot whose window controls match by d
template <bool WC>
__device__ __forceinline__ void phase_all(double2 (&v)[NS], double2 d, uint32_t wm, uint32_t wv)
{
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if (WC && ((k & wm) != wv)) continue;
        v[k] = cmul(v[k], d);
    }
}

template <int RB>
__device__ __forceinline__ void dense_any(double2 (&v)[NS], const GOp &op)
{
    if (op.wm) dense_rb<RB, true>(v, op);
    else dense_rb<RB, false>(v, op);
}

template <int RB>
__device__ __forceinline__ void diag_any(double2 (&v)[NS], const GOp &op)
{
    const bool one = op.u[0].x == 1.0 && op.u[0].y == 0.0;
    if (op.wm) {
        if (one) diag_rb<RB, true, true>(v, op);
        else diag_rb<RB, true, false>(v, op);
    } else {
        if (one) diag_rb<RB, false, true>(v, op);
        else diag_rb<RB, false, false>(v, op);
    }
}

// dense 2x2 on register bit RB where register bit CB == CV (one window control)
template <int RB, int CB, int CV>
__device__ __forceinline__ void cdense_rb(double2 (&v)[NS], const GOp &op)
{
    const double2 u0 = op.u[0], u1 = op.u[1], u2 = op.u[2], u3 = op.u[3];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if (k & (1 << RB)) continue;
        if (((k >> CB) & 1) != CV) continue;
        const double2 x = v[k], y = v[k | (1 << RB)];
        v[k] = cfma2(u0, x, u1, y);
        v[k | (1 << RB)] = cfma2(u2, x, u3, y);
    }
}

// two 2x2 on register bit RB, selected by register bit CS (u[0..3] / u[4..7])
template <int RB, int CS>
__device__ __forceinline__ void dense2_rb(double2 (&v)[NS], const GOp &op)
{
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if (k & (1 << RB)) continue;
        const int o = ((k >> CS) & 1) * 4;
        const double2 x = v[k], y = v[k | (1 << RB)];
        v[k] = cfma2(op.u[o], x, op.u[o + 1], y);
        v[k | (1 << RB)] = cfma2(op.u[o + 2], x, op.u[o + 3], y);
    }
}

#define QS_CD(RB, CB)                                                  \
    case (RB) * 8 + (CB) * 2 + 0: cdense_rb<RB, CB, 0>(v, op); break; \
    case (RB) * 8 + (CB) * 2 + 1: cdense_rb<RB, CB, 1>(v, op); break;
#define QS_D2(RB, CS) \
    case (RB) * 4 + (CS): dense2_rb<RB, CS>(v, op); break;

// Apply ops [i0, i1) of a gate-list pass to the 16 register slots of a thread
// (thread part tpart of the tile index, tile id T).  The op list lives in the
// kernel parameters: every field read is warp-uniform.
__device__ __forceinline__ void run_ops(double2 (&v)[NS], const GOp *ops, int i0, int i1, uint64_t T, uint32_t tpart)
{
    for (int i = i0; i < i1; ++i) {
        const GOp &op = ops[i];
        if ((T & op.fm) != op.fv) continue;           // fixed-bit controls (uniform)
        if ((tpart & op.tm) != op.tv) continue;       // thread-part controls
        switch (op.kind) {
        case GOP_DENSE:
            switch (op.rb) {
            case 0: dense_any<0>(v, op); break;
            case 1: dense_any<1>(v, op); break;
            case 2: dense_any<2>(v, op); break;
            default: dense_any<3>(v, op); break;
            }
            break;
        case GOP_CDENSE:
            switch (op.rb * 8 + op.cs * 2 + op.cv) {
                QS_CD(0, 1) QS_CD(0, 2) QS_CD(0, 3)
                QS_CD(1, 0) QS_CD(1, 2) QS_CD(1, 3)
                QS_CD(2, 0) QS_CD(2, 1) QS_CD(2, 3)
                QS_CD(3, 0) QS_CD(3, 1) QS_CD(3, 2)
            default: break;
            }
            break;
        case GOP_DENSE2:
            switch (op.rb * 4 + op.cs) {
                QS_D2(0, 1) QS_D2(0, 2) QS_D2(0, 3)
                QS_D2(1, 0) QS_D2(1, 2) QS_D2(1, 3)
                QS_D2(2, 0) QS_D2(2, 1) QS_D2(2, 3)
                QS_D2(3, 0) QS_D2(3, 1) QS_D2(3, 2)
            default: break;
            }
            break;
        case GOP_DIAGW:
            switch (op.rb) {
            case 0: diag_any<0>(v, op); break;
            case 1: diag_any<1>(v, op); break;
            case 2: diag_any<2>(v, op); break;
            default: diag_any<3>(v, op); break;
            }
            break;
        default: {
            double2 d;
            if (op.kind == GOP_DIAGT) d = (tpart & op.tb) ? op.u[3] : op.u[0];
            else if (op.kind == GOP_DIAGF) d = ((T >> op.fbit) & 1u) ? op.u[3] : op.u[0];
            else d = op.u[3];
            if (!(d.x == 1.0 && d.y == 0.0)) {
                if (op.wm) phase_all<true>(v, d, op.wm, op.wv);
                else phase_all<false>(v, d, op.wm, op.wv);
            }
        }
        }
    }
}
#undef QS_CD
#undef QS_D2

}  // namespace tile
}  // namespace qs
