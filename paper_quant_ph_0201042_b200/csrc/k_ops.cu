// k_ops.cu -- fused gate-list pass (sm_100a): a run of queued 2x2 gates
// (dense, controlled, diagonal) applied to every
// tile of the shard in one HBM read + write.
//
// The host (api.cu, flush_queue) packs queued gates into passes: every
// non-diagonal gate of a pass targets a "tile" qubit (<= 12 tile bits incl.
// passive low positions), controls may sit anywhere (tile bits: per
// amplitude; other local bits: per tile; rank bits: resolved on the host),
// diagonal gates may act on any local bit.  Gate order is preserved up to
// commutation of gates on disjoint qubits.  Inside a tile, each thread holds
// 16 amplitudes = a 4-bit register window; the op list is cut into segments
// whose non-diagonal targets lie in the segment's window, with an
// XOR-swizzled shared-memory transpose between segments.  The pair update is
// the paper's in-place rule (both rows of a pair in one thread's registers).
#include "qsim_internal.h"
#include "tile_common.cuh"

namespace qs {

namespace {

using namespace tile;

__global__ void __launch_bounds__(256, 1) k_ops_pass(const __grid_constant__ OpsLaunch L, const double2 *in,
                                                     double2 *out, uint64_t ntiles)
{
    extern __shared__ double2 tile_buf[];
    const OpsPass &P = L.P;
    const uint32_t tid = threadIdx.x;
    const int tb = P.tbits - kRegBits;

    const TileMap &m0 = P.seg[0].map;
    const TileMap &mL = P.seg[P.nseg - 1].map;
    uint64_t tin = 0, tout = 0;
    for (int t = 0; t < tb; ++t) {
        const uint64_t bit = (tid >> t) & 1u;
        tin |= bit << P.in_pos[m0.order[t]];
        tout |= bit << P.in_pos[mL.order[t]];
    }
    uint64_t pin[kRegBits], pout[kRegBits];
#pragma unroll
    for (int b = 0; b < kRegBits; ++b) {
        pin[b] = 1ull << P.in_pos[m0.win[b]];
        pout[b] = 1ull << P.in_pos[mL.win[b]];
    }

    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        uint64_t ib = 0;
        for (int f = 0; f < P.nfix; ++f) ib |= ((T >> f) & 1u) << P.fin_pos[f];
        double2 v[NS];
        {
            uint64_t o[NS];
            o[0] = ib | tin;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] | pin[b];
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = in[o[k]];
        }
        uint32_t prev_tpart = 0, prev_stp = 0;
        uint32_t prev_wswz[kRegBits] = {0, 0, 0, 0};
        for (int s = 0; s < P.nseg; ++s) {
            const OpsSeg &sg = P.seg[s];
            const uint32_t tpart = thread_part(sg.map, tb, tid);
            const uint32_t stp = swz(tpart);
            uint32_t wb[kRegBits], wsw[kRegBits];
#pragma unroll
            for (int b = 0; b < kRegBits; ++b) {
                wb[b] = 1u << sg.map.win[b];
                wsw[b] = swz(wb[b]);
            }
            if (s > 0) {
                uint32_t o[NS];
                o[0] = prev_stp;
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                    for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] ^ prev_wswz[b];
                __syncthreads();
#pragma unroll
                for (int k = 0; k < NS; ++k) tile_buf[o[k]] = v[k];
                o[0] = stp;
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                    for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] ^ wsw[b];
                __syncthreads();
#pragma unroll
                for (int k = 0; k < NS; ++k) v[k] = tile_buf[o[k]];
            }
            run_ops(v, L.ops, sg.op_begin, sg.op_end, T, tpart);
            prev_tpart = tpart;
            prev_stp = stp;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b) prev_wswz[b] = wsw[b];
        }
        (void)prev_tpart;
        {
            uint64_t o[NS];
            o[0] = ib | tout;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] | pout[b];
            if (P.nseg == 1) {
                // the gather and scatter maps coincide: each thread rewrites its own addresses
            }
#pragma unroll
            for (int k = 0; k < NS; ++k) out[o[k]] = v[k];
        }
        __syncthreads();   // the tile buffer is reused by the next tile
    }
}

}  // namespace

void launch_ops_pass(Handle *h, const OpsLaunch &L)
{
    if (launch_ops_pass_tma(h, L)) return;
    const OpsPass &P = L.P;
    const size_t smem = (sizeof(double2) << P.tbits);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ops_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double2) << kTileMaxBits));
        attr = true;
    }
    const int threads = 1 << (P.tbits - kRegBits);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ops_pass, threads, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t ntiles = 1ull << P.nfix;
    const uint64_t cap = (uint64_t)h->num_sms * per_sm;
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    prof_begin(h);
    k_ops_pass<<<grid, threads, smem, h->stream>>>(L, h->psi, h->psi, ntiles);
    prof_end(h, "k_ops_pass", (1ull << (P.tbits + P.nfix)) * 32);
}

}  // namespace qs
