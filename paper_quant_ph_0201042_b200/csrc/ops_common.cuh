// ops_common.cuh -- device side of the fused gate-list passes (k_ops.cu:
// direct gather, k_tma.cu: TMA ring): op interpretation on a thread's 32
// register slots and the segment loop with its shared-memory transposes.
#pragma once
#include "qsim_internal.h"
#include "tile_common.cuh"

namespace qs {
namespace ops {

constexpr int RB5 = kOpsRegBits;            // window bits
constexpr int NS5 = 1 << RB5;               // slots per thread
constexpr int kOpsThreads = 1 << (kTileMaxBits - RB5);

using tile::cmul;
using tile::swz;

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

// (x, y) <- (u0 x + u1 y, u2 x + u3 y) in place.  Written in PTX with in-out
// operands so the results land in the slots' own registers: the op
// interpreter joins every op's code path at the loop head, and a result left
// in a temporary costs a register move per double there (the compiler cannot
// overwrite x while y' still needs it; here the y parts of both outputs are
// formed first, then y', then x' with x read by the instruction that
// overwrites it).  16 FP64 instructions, as in cfma2.
__device__ __forceinline__ void pair_inplace(double2 &x, double2 &y, double2 u0, double2 u1, double2 u2, double2 u3)
{
    asm("{\n\t.reg .f64 tr, ti, sr, si, ir, ii, q;\n\t"
        "mul.rn.f64 tr, %6, %2;\n\t"
        "neg.f64 q, %7;\n\t"
        "fma.rn.f64 tr, q, %3, tr;\n\t"
        "mul.rn.f64 ti, %6, %3;\n\t"
        "fma.rn.f64 ti, %7, %2, ti;\n\t"
        "mul.rn.f64 sr, %10, %2;\n\t"
        "neg.f64 q, %11;\n\t"
        "fma.rn.f64 sr, q, %3, sr;\n\t"
        "mul.rn.f64 si, %10, %3;\n\t"
        "fma.rn.f64 si, %11, %2, si;\n\t"
        "fma.rn.f64 %2, %8, %0, sr;\n\t"
        "neg.f64 q, %9;\n\t"
        "fma.rn.f64 %2, q, %1, %2;\n\t"
        "fma.rn.f64 %3, %8, %1, si;\n\t"
        "fma.rn.f64 %3, %9, %0, %3;\n\t"
        "neg.f64 q, %5;\n\t"
        "fma.rn.f64 ir, q, %1, tr;\n\t"
        "fma.rn.f64 ii, %5, %0, ti;\n\t"
        "fma.rn.f64 %0, %4, %0, ir;\n\t"
        "fma.rn.f64 %1, %4, %1, ii;\n\t"
        "}"
        : "+d"(x.x), "+d"(x.y), "+d"(y.x), "+d"(y.y)
        : "d"(u0.x), "d"(u0.y), "d"(u1.x), "d"(u1.y), "d"(u2.x), "d"(u2.y), "d"(u3.x), "d"(u3.y));
}

// x <- d x in place (see pair_inplace)
__device__ __forceinline__ void cmul_inplace(double2 &x, double2 d)
{
    asm("{\n\t.reg .f64 t, u, q;\n\t"
        "mul.rn.f64 t, %3, %1;\n\t"
        "mul.rn.f64 u, %3, %0;\n\t"
        "neg.f64 q, t;\n\t"
        "fma.rn.f64 %0, %2, %0, q;\n\t"
        "fma.rn.f64 %1, %2, %1, u;\n\t"
        "}"
        : "+d"(x.x), "+d"(x.y)
        : "d"(d.x), "d"(d.y));
}

// dense 2x2 (u0 u1; u2 u3) on window bit B for every slot pair whose window
// controls (wm, wv) match
template <int B, bool WC>
__device__ __forceinline__ void dense_rb(double2 (&v)[NS5], double2 u0, double2 u1, double2 u2, double2 u3,
                                         uint32_t wm, uint32_t wv)
{
#pragma unroll
    for (int k = 0; k < NS5; ++k) {
        if (k & (1 << B)) continue;
        if (WC && ((k & wm) != wv)) continue;
        pair_inplace(v[k], v[k | (1 << B)], u0, u1, u2, u3);
    }
}

// dense 2x2 on window bit B where window bit C == CV (one window control)
template <int B, int C, int CV>
__device__ __forceinline__ void cdense_rb(double2 (&v)[NS5], double2 u0, double2 u1, double2 u2, double2 u3)
{
#pragma unroll
    for (int k = 0; k < NS5; ++k) {
        if (k & (1 << B)) continue;
        if (((k >> C) & 1) != CV) continue;
        pair_inplace(v[k], v[k | (1 << B)], u0, u1, u2, u3);
    }
}

// two 2x2 on window bit B selected by window bit C (u[0..3] where it is 0, u[4..7] where 1)
template <int B, int C>
__device__ __forceinline__ void dense2_rb(double2 (&v)[NS5], const GOp &op)
{
    // the pairs with selector 0, then those with selector 1: one matrix live at a time
    {
        const double2 a0 = op.u[0], a1 = op.u[1], a2 = op.u[2], a3 = op.u[3];
#pragma unroll
        for (int k = 0; k < NS5; ++k) {
            if ((k & (1 << B)) || ((k >> C) & 1)) continue;
            pair_inplace(v[k], v[k | (1 << B)], a0, a1, a2, a3);
        }
    }
    {
        const double2 b0 = op.u[4], b1 = op.u[5], b2 = op.u[6], b3 = op.u[7];
#pragma unroll
        for (int k = 0; k < NS5; ++k) {
            if ((k & (1 << B)) || !((k >> C) & 1)) continue;
            pair_inplace(v[k], v[k | (1 << B)], b0, b1, b2, b3);
        }
    }
}

// diag(d0, d1) on window bit B (D0ONE: d0 == 1, only the b = 1 half moves)
template <int B, bool WC, bool D0ONE>
__device__ __forceinline__ void diag_rb(double2 (&v)[NS5], double2 d0, double2 d1, uint32_t wm, uint32_t wv)
{
#pragma unroll
    for (int k = 0; k < NS5; ++k) {
        if (WC && ((k & wm) != wv)) continue;
        if (k & (1 << B)) cmul_inplace(v[k], d1);
        else if (!D0ONE) cmul_inplace(v[k], d0);
    }
}

template <bool WC>
__device__ __forceinline__ void phase_all(double2 (&v)[NS5], double2 d, uint32_t wm, uint32_t wv)
{
#pragma unroll
    for (int k = 0; k < NS5; ++k) {
        if (WC && ((k & wm) != wv)) continue;
        cmul_inplace(v[k], d);
    }
}

#define QS_RB5(BASE, F)                        \
    case (BASE) + 0: F(0); break;              \
    case (BASE) + 1: F(1); break;              \
    case (BASE) + 2: F(2); break;              \
    case (BASE) + 3: F(3); break;              \
    case (BASE) + 4: F(4); break;
#define QS_CD(B, C)                                                                              \
    case OPC_CDENSE + (B) * 10 + (C) * 2 + 0: cdense_rb<B, C, 0>(v, u0, u1, u2, u3); break;    \
    case OPC_CDENSE + (B) * 10 + (C) * 2 + 1: cdense_rb<B, C, 1>(v, u0, u1, u2, u3); break;
#define QS_D2(B, C) \
    case OPC_DENSE2 + (B) * 5 + (C): dense2_rb<B, C>(v, op); break;
#define QS_DW(B)                                                                                   \
    case OPC_DIAGW + (B) * 4 + 0: diag_rb<B, false, false>(v, op.u[0], op.u[3], 0, 0); break;       \
    case OPC_DIAGW + (B) * 4 + 1: diag_rb<B, false, true>(v, op.u[0], op.u[3], 0, 0); break;        \
    case OPC_DIAGW + (B) * 4 + 2: diag_rb<B, true, false>(v, op.u[0], op.u[3], op.wm, op.wv); break; \
    case OPC_DIAGW + (B) * 4 + 3: diag_rb<B, true, true>(v, op.u[0], op.u[3], op.wm, op.wv); break;
#define QS_DN(B) dense_rb<B, false>(v, u0, u1, u2, u3, 0, 0)
#define QS_DNW(B) dense_rb<B, true>(v, u0, u1, u2, u3, op.wm, op.wv)

// One op on the 32 register slots of a thread (thread part tpart of the tile
// index, tile id T).  Every field of op is warp-uniform; code = op.code,
// fetched by the caller one op ahead, selects the case in one indexed branch.
__device__ __forceinline__ void apply_op(double2 (&v)[NS5], const GOp &op, uint32_t code, uint64_t T, uint32_t tpart,
                                         uint32_t traj)
{
    if ((code & kOpChkFixed) && (T & op.fm) != op.fv) return;          // fixed-bit controls
    if ((code & kOpChkThread) && (tpart & op.tm) != op.tv) return;     // thread-part controls
    const uint32_t c = code & 0xffu;
    if (c < OPC_DENSE2) {
        // dense forms: the matrix (u[4..7] where the selector is 1; DENSET: this
        // tile's trajectory matrix, one uniform 64-byte load, L1-cached)
        const double2 *m = op.u;
        if (code & kOpTraj) m = op.tab + 4 * (uint64_t)traj;
        else if ((code & kOpSel) &&
                 ((tpart & op.tsel) != 0 || (op.fsel != 0xffu && ((T >> op.fsel) & 1u))))
            m = op.u + 4;
        const double2 u0 = m[0], u1 = m[1], u2 = m[2], u3 = m[3];
        switch (c) {
            QS_RB5(OPC_DENSE, QS_DN)
            QS_RB5(OPC_DENSE + 5, QS_DNW)
            QS_CD(0, 1) QS_CD(0, 2) QS_CD(0, 3) QS_CD(0, 4)
            QS_CD(1, 0) QS_CD(1, 2) QS_CD(1, 3) QS_CD(1, 4)
            QS_CD(2, 0) QS_CD(2, 1) QS_CD(2, 3) QS_CD(2, 4)
            QS_CD(3, 0) QS_CD(3, 1) QS_CD(3, 2) QS_CD(3, 4)
            QS_CD(4, 0) QS_CD(4, 1) QS_CD(4, 2) QS_CD(4, 3)
        default: break;
        }
        return;
    }
    switch (c) {
        QS_D2(0, 1) QS_D2(0, 2) QS_D2(0, 3) QS_D2(0, 4)
        QS_D2(1, 0) QS_D2(1, 2) QS_D2(1, 3) QS_D2(1, 4)
        QS_D2(2, 0) QS_D2(2, 1) QS_D2(2, 3) QS_D2(2, 4)
        QS_D2(3, 0) QS_D2(3, 1) QS_D2(3, 2) QS_D2(3, 4)
        QS_D2(4, 0) QS_D2(4, 1) QS_D2(4, 2) QS_D2(4, 3)
        QS_DW(0) QS_DW(1) QS_DW(2) QS_DW(3) QS_DW(4)
    default: {
        const uint32_t kind = op.kind;
        double2 d;
        if (kind == GOP_DIAGT) d = (tpart & op.tb) ? op.u[3] : op.u[0];
        else if (kind == GOP_DIAGF) d = ((T >> op.fbit) & 1u) ? op.u[3] : op.u[0];
        else d = op.u[3];
        if (!(d.x == 1.0 && d.y == 0.0)) {
            if (op.wm) phase_all<true>(v, d, op.wm, op.wv);
            else phase_all<false>(v, d, op.wm, op.wv);
        }
    } break;
    }
}
#undef QS_RB5
#undef QS_DW
#undef QS_DN
#undef QS_DNW
#undef QS_CD
#undef QS_D2

// DENSE on window bit rb (case OPC_DENSE + rb) or DENSE2 (OPC_DENSE2 + rb * 5
// + cs) with no control checks, trajectory table or run-time selector
__device__ __forceinline__ void apply_dense_fast(double2 (&v)[NS5], const GOp &op, uint32_t c)
{
    if (c < OPC_DENSE + 5) {
        const double2 u0 = op.u[0], u1 = op.u[1], u2 = op.u[2], u3 = op.u[3];
        switch (c) {
        case 0: dense_rb<0, false>(v, u0, u1, u2, u3, 0, 0); break;
        case 1: dense_rb<1, false>(v, u0, u1, u2, u3, 0, 0); break;
        case 2: dense_rb<2, false>(v, u0, u1, u2, u3, 0, 0); break;
        case 3: dense_rb<3, false>(v, u0, u1, u2, u3, 0, 0); break;
        default: dense_rb<4, false>(v, u0, u1, u2, u3, 0, 0); break;
        }
        return;
    }
    switch (c) {
#define QS_F2(B, C) \
    case OPC_DENSE2 + (B) * 5 + (C): dense2_rb<B, C>(v, op); break;
        QS_F2(0, 1) QS_F2(0, 2) QS_F2(0, 3) QS_F2(0, 4)
        QS_F2(1, 0) QS_F2(1, 2) QS_F2(1, 3) QS_F2(1, 4)
        QS_F2(2, 0) QS_F2(2, 1) QS_F2(2, 3) QS_F2(2, 4)
        QS_F2(3, 0) QS_F2(3, 1) QS_F2(3, 2) QS_F2(3, 4)
        QS_F2(4, 0) QS_F2(4, 1) QS_F2(4, 2) QS_F2(4, 3)
#undef QS_F2
    default: break;
    }
}

__device__ __forceinline__ uint32_t seg_thread_part(const OpsSeg &s, int tb, uint32_t tid)
{
    uint32_t ti = 0;
    for (int t = 0; t < tb; ++t) ti |= ((tid >> t) & 1u) << s.order[t];
    return ti;
}


// The segments of one tile: v holds the tile in segment 0's register map on
// entry and in the last segment's map on exit; buf (2^tbits double2, shared)
// carries the transposes between register windows.
// barrier over the threads that share one tile buffer: the whole CTA, or one
// 128-thread warpgroup (named barrier 1 + wg) in the ping-pong kernel
struct CtaSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct WgSync {
    uint32_t id;
    __device__ __forceinline__ void operator()() const
    {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kOpsThreads) : "memory");
    }
};

template <class Sync = CtaSync>
__device__ __forceinline__ void run_segments(double2 (&v)[NS5], const OpsLaunch &L, uint64_t T, uint32_t tid, int tb,
                                             double2 *buf, Sync sync = Sync(), const GOp *ops = nullptr,
                                             const uint32_t *tparts = nullptr)
{
    const OpsPass &P = L.P;
    uint32_t traj = P.bat_rank;
    for (int i = 0; i < P.nbat; ++i) traj |= (uint32_t)((T >> P.bat_fix[i]) & 1u) << P.bat_sh[i];
    uint32_t prev_stp = 0;
    uint32_t prev_wsw[RB5] = {0, 0, 0, 0, 0};
    for (int s = 0; s < P.nseg; ++s) {
        const OpsSeg &sg = P.seg[s];
        // thread part of the tile index: precomputed per segment (shared memory) or here
        const uint32_t tpart = tparts ? tparts[(s << (kTileMaxBits - RB5)) + tid] : seg_thread_part(sg, tb, tid);
        const uint32_t stp = swz(tpart);
        uint32_t wsw[RB5];
#pragma unroll
        for (int b = 0; b < RB5; ++b) wsw[b] = swz(1u << sg.win[b]);
        if (s > 0) {
            sync();   // previous readers of the tile buffer are done
#pragma unroll
            for (int k = 0; k < NS5; ++k) {
                uint32_t o = prev_stp;
#pragma unroll
                for (int b = 0; b < RB5; ++b)
                    if (k & (1 << b)) o ^= prev_wsw[b];
                buf[o] = v[k];
            }
            sync();
#pragma unroll
            for (int k = 0; k < NS5; ++k) {
                uint32_t o = stp;
#pragma unroll
                for (int b = 0; b < RB5; ++b)
                    if (k & (1 << b)) o ^= wsw[b];
                v[k] = buf[o];
            }
        }
        // the next op's dispatch word is fetched while this op runs
        const GOp *OP = ops ? ops : L.ops;   // a shared-memory copy of the op list, or the parameters
        uint32_t code = sg.op_begin < sg.op_end ? OP[sg.op_begin].code : 0u;
        for (int i = sg.op_begin; i < sg.op_end; ++i) {
            const uint32_t c = code;
            if (i + 1 < sg.op_end) code = OP[i + 1].code;
            if (c < OPC_DENSE + 5 || (c >= OPC_DENSE2 && c < OPC_DIAGW)) {
                // fast path (noisy circuits: almost every op): a dense 2x2, or a
                // pair of them selected by a window bit, with no run-time checks
                apply_dense_fast(v, OP[i], c);
            } else {
                apply_op(v, OP[i], c, T, tpart, traj);
            }
        }
        prev_stp = stp;
#pragma unroll
        for (int b = 0; b < RB5; ++b) prev_wsw[b] = wsw[b];
    }
}

}  // namespace ops
}  // namespace qs
