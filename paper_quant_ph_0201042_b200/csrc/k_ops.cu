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
#include <cstdlib>

#include "ops_common.cuh"

namespace qs {

namespace {

using namespace ops;

// segments whose thread parts are precomputed in shared memory (more: computed per tile)
constexpr int kOpsPreSegs = 12;

__global__ void __launch_bounds__(kOpsThreads, 2) k_ops_pass(const __grid_constant__ OpsLaunch L, double2 *psi,
                                                             uint64_t ntiles)
{
    extern __shared__ double2 tile_buf[];
    const OpsPass &P = L.P;
    const uint32_t tid = threadIdx.x;
    // the op list in shared memory: indexed constant loads of a ~24 KB
    // parameter block miss the constant cache (~16% measured), an LDS does not
    GOp *ops = reinterpret_cast<GOp *>(tile_buf + ((size_t)1 << P.tbits));
    // per-tile index arithmetic from tables built once: the fixed-bit part of
    // a tile's offset byte by byte, and every segment's thread part
    uint64_t *ibtab = reinterpret_cast<uint64_t *>(ops + P.nops);   // [4][256]
    uint32_t *tparts = reinterpret_cast<uint32_t *>(ibtab + 4 * 256);
    const bool pre_tp = P.nseg <= kOpsPreSegs;
    const int tb = P.tbits - RB5;
    {
        const int4 *src = reinterpret_cast<const int4 *>(L.ops);
        int4 *dst = reinterpret_cast<int4 *>(ops);
        const int words = P.nops * (int)(sizeof(GOp) / sizeof(int4));
        for (int w = tid; w < words; w += blockDim.x) dst[w] = src[w];
        for (int e = tid; e < 4 * 256; e += blockDim.x) {
            const int k = e >> 8, x = e & 255;
            uint64_t o = 0;
            for (int j = 0; j < 8; ++j) {
                const int f = 8 * k + j;
                if (f < P.nfix && ((x >> j) & 1)) o |= 1ull << P.fin_pos[f];
            }
            ibtab[e] = o;
        }
        if (pre_tp)
            for (int s = 0; s < P.nseg; ++s) tparts[(s << (kTileMaxBits - RB5)) + tid] = seg_thread_part(P.seg[s], tb, tid);
        __syncthreads();
    }

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
        const uint64_t ib = ibtab[T & 255] | ibtab[256 + ((T >> 8) & 255)] | ibtab[512 + ((T >> 16) & 255)] |
                            ibtab[768 + ((T >> 24) & 255)];
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
        run_segments(v, L, T, tid, tb, tile_buf, CtaSync(), ops, pre_tp ? tparts : nullptr);
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
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const OpsPass &P = L.P;
    // memory-bound passes (little FP64 work per amplitude) stream best through
    // the TMA ring; FP64-bound ones through two CTAs per SM (k_ops_pass)
    static const double tma_max = std::getenv("QSIM_OPS_TMA_MAX") ? std::atof(std::getenv("QSIM_OPS_TMA_MAX")) : 4.0;
    double cost = 0;
    for (int i = 0; i < P.nops; ++i) {
        const GOp &g = L.ops[i];
        double c = (g.kind == GOP_DENSE || g.kind == GOP_DENSE2 || g.kind == GOP_DENSET) ? 1.0 : 0.5;
        if (g.fm) c *= 0.5;
        cost += c;
    }
    if (cost <= tma_max && launch_ops_pass_tma(h, L)) return;
    // FP64 work beyond the TMA ring's: the ping-pong TMA kernel overlaps loads
    // with both warpgroups' arithmetic (configs[3]'s 9-gate H passes: 11.9 ->
    // 10.6 ms; configs[4]'s 25-gate passes 7% faster than k_ops_pass once both
    // read the op list from shared memory); tiles that are not a <= 5-D TMA
    // box go to k_ops_pass
    static const double pp_max = std::getenv("QSIM_OPS_PP_MAX") ? std::atof(std::getenv("QSIM_OPS_PP_MAX")) : 1e9;
    if (cost <= pp_max && launch_ops_pass_pp(h, L)) return;
    const size_t pre = (P.nseg <= kOpsPreSegs ? (size_t)P.nseg << (kTileMaxBits - RB5) : 0) * sizeof(uint32_t);
    const size_t smem = (sizeof(double2) << P.tbits) + (size_t)P.nops * sizeof(GOp) + 4 * 256 * sizeof(uint64_t) + pre;
    static uint64_t attr = 0;
    if (first_use_on_device(attr)) {
        cudaFuncSetAttribute(k_ops_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((sizeof(double2) << kTileMaxBits) + kOpsParam * sizeof(GOp) +
                                   4 * 256 * sizeof(uint64_t) +
                                   ((size_t)kOpsPreSegs << (kTileMaxBits - RB5)) * sizeof(uint32_t)));
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
