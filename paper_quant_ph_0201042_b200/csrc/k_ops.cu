// k_ops.cu -- fused gate-list pass (sm_100a): a run of queued 2x2 gates
// (dense, controlled, diagonal) applied to every
// tile of the shard in one HBM read + write.
//
// The host planner (plan_ops.cu) packs queued gates into passes and orders
// each pass into "segments": a tile is 2^tbits amplitudes (<= 4096), each of
// the 2^(tbits-5) threads holds 32 of them in registers = a 5-bit register
// window of tile bits; a segment's gates all act non-diagonally on window
// bits only, so a pair update is the paper's in-place rule (PAPER.md:329-337,
// both rows of a pair in one thread's registers, no barrier).  Between
// segments the tile goes through shared memory once (XOR-swizzled transpose)
// to bring the next window into registers.
//
// Noisy circuits make this pass FP64-bound (8 FMA-class instructions per
// amplitude per dense gate vs 32 bytes of HBM traffic per amplitude per
// pass), so the kernel is built for the FP64 pipe: 32 slots per thread give
// 16 independent pair updates per op, two 128-thread CTAs per SM overlap one
// CTA's gather / transposes with the other's arithmetic, and every op
// parameter is a warp-uniform constant-bank read (the op list travels in the
// kernel parameters).
#include "qsim_internal.h"
#include "tile_common.cuh"

namespace qs {

namespace {

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
        const double2 x = v[k], y = v[k | (1 << B)];
        v[k] = cfma2(u0, x, u1, y);
        v[k | (1 << B)] = cfma2(u2, x, u3, y);
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
        const double2 x = v[k], y = v[k | (1 << B)];
        v[k] = cfma2(u0, x, u1, y);
        v[k | (1 << B)] = cfma2(u2, x, u3, y);
    }
}

// two 2x2 on window bit B selected by window bit C (u[0..3] where it is 0, u[4..7] where 1)
template <int B, int C>
__device__ __forceinline__ void dense2_rb(double2 (&v)[NS5], const GOp &op)
{
    const double2 a0 = op.u[0], a1 = op.u[1], a2 = op.u[2], a3 = op.u[3];
    const double2 b0 = op.u[4], b1 = op.u[5], b2 = op.u[6], b3 = op.u[7];
#pragma unroll
    for (int k = 0; k < NS5; ++k) {
        if (k & (1 << B)) continue;
        const bool s = (k >> C) & 1;
        const double2 x = v[k], y = v[k | (1 << B)];
        v[k] = cfma2(s ? b0 : a0, x, s ? b1 : a1, y);
        v[k | (1 << B)] = cfma2(s ? b2 : a2, x, s ? b3 : a3, y);
    }
}

// diag(d0, d1) on window bit B (D0ONE: d0 == 1, only the b = 1 half moves)
template <int B, bool WC, bool D0ONE>
__device__ __forceinline__ void diag_rb(double2 (&v)[NS5], double2 d0, double2 d1, uint32_t wm, uint32_t wv)
{
#pragma unroll
    for (int k = 0; k < NS5; ++k) {
        if (WC && ((k & wm) != wv)) continue;
        if (k & (1 << B)) v[k] = cmul(v[k], d1);
        else if (!D0ONE) v[k] = cmul(v[k], d0);
    }
}

template <bool WC>
__device__ __forceinline__ void phase_all(double2 (&v)[NS5], double2 d, uint32_t wm, uint32_t wv)
{
#pragma unroll
    for (int k = 0; k < NS5; ++k) {
        if (WC && ((k & wm) != wv)) continue;
        v[k] = cmul(v[k], d);
    }
}

template <int B>
__device__ __forceinline__ void dense_any(double2 (&v)[NS5], double2 u0, double2 u1, double2 u2, double2 u3,
                                          uint32_t wm, uint32_t wv)
{
    if (wm) dense_rb<B, true>(v, u0, u1, u2, u3, wm, wv);
    else dense_rb<B, false>(v, u0, u1, u2, u3, 0, 0);
}

template <int B>
__device__ __forceinline__ void diag_any(double2 (&v)[NS5], double2 d0, double2 d1, uint32_t wm, uint32_t wv)
{
    const bool one = d0.x == 1.0 && d0.y == 0.0;
    if (wm) {
        if (one) diag_rb<B, true, true>(v, d0, d1, wm, wv);
        else diag_rb<B, true, false>(v, d0, d1, wm, wv);
    } else {
        if (one) diag_rb<B, false, true>(v, d0, d1, 0, 0);
        else diag_rb<B, false, false>(v, d0, d1, 0, 0);
    }
}

#define QS_CD(B, C)                                                            \
    case (B) * 16 + (C) * 2 + 0: cdense_rb<B, C, 0>(v, u0, u1, u2, u3); break; \
    case (B) * 16 + (C) * 2 + 1: cdense_rb<B, C, 1>(v, u0, u1, u2, u3); break;
#define QS_D2(B, C) \
    case (B) * 8 + (C): dense2_rb<B, C>(v, op); break;

// One op on the 32 register slots of a thread (thread part tpart of the tile
// index, tile id T).  Every field of op is warp-uniform.
__device__ __forceinline__ void apply_op(double2 (&v)[NS5], const GOp &op, uint64_t T, uint32_t tpart)
{
    if ((T & op.fm) != op.fv) return;           // fixed-bit controls (uniform)
    if ((tpart & op.tm) != op.tv) return;       // thread-part controls
    const uint32_t kind = op.kind;
    if (kind == GOP_DENSE || kind == GOP_CDENSE) {
        // matrix u[4..7] where the selector (thread bit tsel or tile-id bit fsel) is 1
        const bool s = (tpart & op.tsel) != 0 || (op.fsel != 0xffu && ((T >> op.fsel) & 1u));
        const int o = s ? 4 : 0;
        const double2 u0 = op.u[o], u1 = op.u[o + 1], u2 = op.u[o + 2], u3 = op.u[o + 3];
        if (kind == GOP_DENSE) {
            switch (op.rb) {
            case 0: dense_any<0>(v, u0, u1, u2, u3, op.wm, op.wv); break;
            case 1: dense_any<1>(v, u0, u1, u2, u3, op.wm, op.wv); break;
            case 2: dense_any<2>(v, u0, u1, u2, u3, op.wm, op.wv); break;
            case 3: dense_any<3>(v, u0, u1, u2, u3, op.wm, op.wv); break;
            default: dense_any<4>(v, u0, u1, u2, u3, op.wm, op.wv); break;
            }
        } else {
            switch (op.rb * 16 + op.cs * 2 + op.cv) {
                QS_CD(0, 1) QS_CD(0, 2) QS_CD(0, 3) QS_CD(0, 4)
                QS_CD(1, 0) QS_CD(1, 2) QS_CD(1, 3) QS_CD(1, 4)
                QS_CD(2, 0) QS_CD(2, 1) QS_CD(2, 3) QS_CD(2, 4)
                QS_CD(3, 0) QS_CD(3, 1) QS_CD(3, 2) QS_CD(3, 4)
                QS_CD(4, 0) QS_CD(4, 1) QS_CD(4, 2) QS_CD(4, 3)
            default: break;
            }
        }
        return;
    }
    if (kind == GOP_DENSE2) {
        switch (op.rb * 8 + op.cs) {
            QS_D2(0, 1) QS_D2(0, 2) QS_D2(0, 3) QS_D2(0, 4)
            QS_D2(1, 0) QS_D2(1, 2) QS_D2(1, 3) QS_D2(1, 4)
            QS_D2(2, 0) QS_D2(2, 1) QS_D2(2, 3) QS_D2(2, 4)
            QS_D2(3, 0) QS_D2(3, 1) QS_D2(3, 2) QS_D2(3, 4)
            QS_D2(4, 0) QS_D2(4, 1) QS_D2(4, 2) QS_D2(4, 3)
        default: break;
        }
        return;
    }
    if (kind == GOP_DIAGW) {
        const double2 d0 = op.u[0], d1 = op.u[3];
        switch (op.rb) {
        case 0: diag_any<0>(v, d0, d1, op.wm, op.wv); break;
        case 1: diag_any<1>(v, d0, d1, op.wm, op.wv); break;
        case 2: diag_any<2>(v, d0, d1, op.wm, op.wv); break;
        case 3: diag_any<3>(v, d0, d1, op.wm, op.wv); break;
        default: diag_any<4>(v, d0, d1, op.wm, op.wv); break;
        }
        return;
    }
    double2 d;
    if (kind == GOP_DIAGT) d = (tpart & op.tb) ? op.u[3] : op.u[0];
    else if (kind == GOP_DIAGF) d = ((T >> op.fbit) & 1u) ? op.u[3] : op.u[0];
    else d = op.u[3];
    if (!(d.x == 1.0 && d.y == 0.0)) {
        if (op.wm) phase_all<true>(v, d, op.wm, op.wv);
        else phase_all<false>(v, d, op.wm, op.wv);
    }
}
#undef QS_CD
#undef QS_D2

__device__ __forceinline__ uint32_t seg_thread_part(const OpsSeg &s, int tb, uint32_t tid)
{
    uint32_t ti = 0;
    for (int t = 0; t < tb; ++t) ti |= ((tid >> t) & 1u) << s.order[t];
    return ti;
}

__global__ void __launch_bounds__(kOpsThreads, 2) k_ops_pass(const __grid_constant__ OpsLaunch L, double2 *psi,
                                                             uint64_t ntiles)
{
    extern __shared__ double2 tile_buf[];
    const OpsPass &P = L.P;
    const uint32_t tid = threadIdx.x;
    const int tb = P.tbits - RB5;

    const OpsSeg &s0 = P.seg[0];
    const OpsSeg &sL = P.seg[P.nseg - 1];
    uint64_t tin = 0, tout = 0;
    for (int t = 0; t < tb; ++t) {
        const uint64_t bit = (tid >> t) & 1u;
        tin |= bit << P.in_pos[s0.order[t]];
        tout |= bit << P.in_pos[sL.order[t]];
    }
    uint64_t pin[RB5], pout[RB5];
#pragma unroll
    for (int b = 0; b < RB5; ++b) {
        pin[b] = 1ull << P.in_pos[s0.win[b]];
        pout[b] = 1ull << P.in_pos[sL.win[b]];
    }

    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        uint64_t ib = 0;
        for (int f = 0; f < P.nfix; ++f) ib |= ((T >> f) & 1u) << P.fin_pos[f];
        double2 v[NS5];
        {
            const uint64_t base = ib | tin;
#pragma unroll
            for (int k = 0; k < NS5; ++k) {
                uint64_t o = base;
#pragma unroll
                for (int b = 0; b < RB5; ++b)
                    if (k & (1 << b)) o |= pin[b];
                v[k] = psi[o];
            }
        }
        uint32_t prev_stp = 0;
        uint32_t prev_wsw[RB5] = {0, 0, 0, 0, 0};
        for (int s = 0; s < P.nseg; ++s) {
            const OpsSeg &sg = P.seg[s];
            const uint32_t tpart = seg_thread_part(sg, tb, tid);
            const uint32_t stp = swz(tpart);
            uint32_t wsw[RB5];
#pragma unroll
            for (int b = 0; b < RB5; ++b) wsw[b] = swz(1u << sg.win[b]);
            if (s > 0) {
                __syncthreads();   // previous readers of the tile buffer are done
#pragma unroll
                for (int k = 0; k < NS5; ++k) {
                    uint32_t o = prev_stp;
#pragma unroll
                    for (int b = 0; b < RB5; ++b)
                        if (k & (1 << b)) o ^= prev_wsw[b];
                    tile_buf[o] = v[k];
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < NS5; ++k) {
                    uint32_t o = stp;
#pragma unroll
                    for (int b = 0; b < RB5; ++b)
                        if (k & (1 << b)) o ^= wsw[b];
                    v[k] = tile_buf[o];
                }
            }
            for (int i = sg.op_begin; i < sg.op_end; ++i) apply_op(v, L.ops[i], T, tpart);
            prev_stp = stp;
#pragma unroll
            for (int b = 0; b < RB5; ++b) prev_wsw[b] = wsw[b];
        }
        {
            const uint64_t base = ib | tout;
#pragma unroll
            for (int k = 0; k < NS5; ++k) {
                uint64_t o = base;
#pragma unroll
                for (int b = 0; b < RB5; ++b)
                    if (k & (1 << b)) o |= pout[b];
                psi[o] = v[k];
            }
        }
        // in place: every tile is read and written by the same CTA, tiles are disjoint
    }
}

}  // namespace

void launch_ops_pass(Handle *h, const OpsLaunch &L)
{
    const OpsPass &P = L.P;
    const size_t smem = sizeof(double2) << P.tbits;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ops_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double2) << kTileMaxBits));
        attr = true;
    }
    const int threads = 1 << (P.tbits - RB5);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ops_pass, threads, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t ntiles = 1ull << P.nfix;
    const uint64_t cap = (uint64_t)h->num_sms * per_sm;
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    prof_begin(h);
    k_ops_pass<<<grid, threads, smem, h->stream>>>(L, h->psi, ntiles);
    prof_end(h, "k_ops_pass", (1ull << (P.tbits + P.nfix)) * 32);
}

}  // namespace qs
