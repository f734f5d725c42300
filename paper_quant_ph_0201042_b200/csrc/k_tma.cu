// k_tma.cu -- TMA-pipelined, warp-specialised fused QFT / H pass (sm_100a).
//
// Same arithmetic as k_tile.cu (tile_body), different data movement:
//   * a persistent CTA per SM (8 warps, 16 amplitudes per thread) streams
//     tiles HBM -> shared memory with one cp.async.bulk.tensor (TMA) per tile
//     into a 3-stage ring of 64 KiB buffers; completion is signalled on an
//     mbarrier (complete_tx::bytes);
//   * the warps read the tile from its TMA box layout, run the register maps
//     (transposes in the same buffer), write the result in the output box
//     layout; thread 0 issues the TMA store (bulk_group), waits until the
//     previous tile's store has read its buffer and immediately refills that
//     buffer with the load of the tile two steps ahead.
// (No separate producer warp: at 224 registers per thread a 9th warp would
// not fit the per-SM-sub-partition register file.)
// So while a tile is being computed, the next two are in flight from HBM and
// the previous one is being written back: the pass streams at HBM speed as
// long as the FP64 + shared-memory work of a tile hides under its transfer
// time.  The tile geometry (which positions form the box) comes from the
// block-move pass plan in api.cu; positions outside the box are coordinates
// of a <= 5-D tensor map (runs of consecutive positions).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "qsim_internal.h"
#include "ops_common.cuh"
#include "tile_common.cuh"
#include "mbar.cuh"
#include "tma_host.h"

namespace qs {

namespace {

using namespace tile;

constexpr int kStages = 3;
constexpr int kTmaTileBits = 12;                          // 4096 amplitudes
constexpr uint32_t kTileBytes = 16u << kTmaTileBits;      // 64 KiB
constexpr int kThreads = 1 << (kTmaTileBits - kRegBits);

struct TmaArgs {
    // per tensor-map dim d (0..4): first tile-id bit and length of the fixed
    // run it addresses (len 0: a box dim, coordinate 0)
    int in_first[5], in_len[5];
    int out_first[5], out_len[5];
    // smem amplitude index of each tile bit in the load / store boxes
    int in_rank[kTileMaxBits], out_rank[kTileMaxBits];
};

__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *map, const int (&c)[5], uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_store(const CUtensorMap *map, const int (&c)[5], const void *src)
{
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                     (uint64_t)map),
                 "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read()
{
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void coords(const int (&first)[5], const int (&len)[5], uint64_t T, int (&c)[5])
{
#pragma unroll
    for (int d = 0; d < 5; ++d)
        c[d] = len[d] ? (int)((T >> first[d]) & ((1ull << len[d]) - 1)) : 0;
}

template <int NM>
__global__ void __launch_bounds__(kThreads, 1)
    k_tile_tma(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
               const __grid_constant__ TilePass tp, const __grid_constant__ TmaArgs ta, uint64_t ntiles)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);                       // kStages x 4096
    double2 *tab = bufs + kStages * (1u << kTmaTileBits);                          // 1024
    uint64_t *full = reinterpret_cast<uint64_t *>(tab + 1024);                     // kStages
    const uint32_t tid = threadIdx.x;
    const double sg = tp.inverse ? -1.0 : 1.0;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t k = tid; k < 1024; k += blockDim.x) {
        double s, c;
        sincospi((double)k / 512.0, &s, &c);
        tab[k] = make_double2(c, sg * s);
    }
    __syncthreads();
    // prologue: the first two tiles of this CTA are requested right away
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&in_map) : "memory");
        for (uint64_t q = 0; q < kStages - 1; ++q) {
            const uint64_t T = blockIdx.x + q * gridDim.x;
            if (T >= ntiles) break;
            int c[5];
            coords(ta.in_first, ta.in_len, T, c);
            mbar_expect_tx(&full[q], kTileBytes);
            tma_load(bufs + (size_t)q * (1u << kTmaTileBits), &in_map, c, &full[q]);
        }
    }

    // ---------------- compute warps
    constexpr int tb = kTmaTileBits - kRegBits;   // 8 thread bits
    uint32_t tpart[NM], stp[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        tpart[m] = thread_part(tp.map[m], tb, tid);
        stp[m] = swz(tpart[m]);
    }
    // box-layout indices: map 0 reads the load box, the last map writes the store box
    uint32_t lin = 0, lout = 0;
    for (int t = 0; t < tb; ++t) {
        lin |= ((tid >> t) & 1u) << ta.in_rank[tp.map[0].order[t]];
        lout |= ((tid >> t) & 1u) << ta.out_rank[tp.map[NM - 1].order[t]];
    }
    uint32_t pin[kRegBits], pout[kRegBits];
#pragma unroll
    for (int b = 0; b < kRegBits; ++b) {
        pin[b] = 1u << ta.in_rank[tp.map[0].win[b]];
        pout[b] = 1u << ta.out_rank[tp.map[NM - 1].win[b]];
    }
    const bool twid = !tp.hadamard_only && tp.a > 0 && (tp.n_et > 0 || tp.n_ef > 0 || tp.y_const != 0);
    const uint32_t amask = (1u << tp.a) - 1u;
    const uint32_t Jt = tp.a > 0 ? (__brev(tpart[0] & amask) >> (32 - tp.a)) : 0u;
    uint64_t yt = 0;
    for (int e = 0; e < tp.n_et; ++e) yt += (uint64_t)((tpart[0] >> tp.et_bit[e]) & 1u) << tp.et_w[e];

    uint64_t j = 0;
    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x, ++j) {
        const int s = (int)(j % kStages);
        double2 *buf = bufs + (size_t)s * (1u << kTmaTileBits);
        mbar_wait(&full[s], (uint32_t)((j / kStages) & 1));
        double2 v[NS];
        {
            uint32_t o[NS];
            o[0] = lin;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] | pin[b];
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = buf[o[k]];
        }
        tile_body<NM, false>(v, tp, tpart, stp, tab, buf, T, yt, Jt, twid, amask, sg);
        {
            uint32_t o[NS];
            o[0] = lout;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] | pout[b];
            tile_sync<false>();   // everybody is done reading this buffer
#pragma unroll
            for (int k = 0; k < NS; ++k) buf[o[k]] = v[k];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tile_sync<false>();
        if (tid == 0) {
            int c[5];
            coords(ta.out_first, ta.out_len, T, c);
            tma_store(&out_map, c, buf);
            // the previous tile's store has finished reading its buffer:
            // refill it with the tile two steps ahead
            bulk_wait_read<1>();
            const uint64_t Tn = T + (uint64_t)(kStages - 1) * gridDim.x;
            if (Tn < ntiles) {
                const int sn = (int)((j + kStages - 1) % kStages);
                coords(ta.in_first, ta.in_len, Tn, c);
                mbar_expect_tx(&full[sn], kTileBytes);
                tma_load(bufs + (size_t)sn * (1u << kTmaTileBits), &in_map, c, &full[sn]);
            }
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Specialised QFT / H pass: the number of active wires A, the direction and
// H-only mode are compile-time, so the register windows, the wires each
// window transforms and the R_1..R_3 rotations are static: no runtime
// branches around the register updates (no phi moves) and the rotation by
// -+i is a free swap/negation.  Window s holds tile bits [w0, w0+4) with
// w0 = 4s, except the last window, which ends at wire A-1 (already
// transformed wires fill it up, so the passive tile bits stay thread bits).
template <int A, bool INV, bool HONLY>
__global__ void __launch_bounds__(kThreads, 1)
    k_qft_tma(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
              const __grid_constant__ TilePass tp, const __grid_constant__ TmaArgs ta, uint64_t ntiles, int gbits)
{
    // this CTA's j-th tile: groups of 2^gbits consecutive tiles (adjacent
    // runs of the lowest fixed positions), groups strided over the grid
    const uint64_t gmask = (1ull << gbits) - 1;
    auto tile_of = [&](uint64_t jj) -> uint64_t {
        return ((blockIdx.x + (jj >> gbits) * (uint64_t)gridDim.x) << gbits) | (jj & gmask);
    };
    static_assert(kRegBits == 4 && kTmaTileBits == 12 && A >= 4 && A <= 10, "window layout");
    constexpr int NST = (A + 3) / 4;   // register windows
    constexpr double SG = INV ? -1.0 : 1.0;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);
    double2 *tab = bufs + kStages * (1u << kTmaTileBits);
    uint64_t *full = reinterpret_cast<uint64_t *>(tab + 1024);
    const uint32_t tid = threadIdx.x;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t k = tid; k < 1024; k += blockDim.x) {
        double sn, cs;
        sincospi((double)k / 512.0, &sn, &cs);
        tab[k] = make_double2(cs, SG * sn);
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&in_map) : "memory");
        for (uint64_t q = 0; q < kStages - 1; ++q) {
            const uint64_t T = tile_of(q);
            if (T >= ntiles) break;
            int c[5];
            coords(ta.in_first, ta.in_len, T, c);
            mbar_expect_tx(&full[q], kTileBytes);
            tma_load(bufs + (size_t)q * (1u << kTmaTileBits), &in_map, c, &full[q]);
        }
    }

    constexpr int tb = kTmaTileBits - kRegBits;
    uint32_t tpart[NST], stp[NST];
#pragma unroll
    for (int m = 0; m < NST; ++m) {
        tpart[m] = thread_part(tp.map[m], tb, tid);
        stp[m] = swz(tpart[m]);
    }
    uint32_t lin = 0, lout = 0;
    for (int t = 0; t < tb; ++t) {
        lin |= ((tid >> t) & 1u) << ta.in_rank[tp.map[0].order[t]];
        lout |= ((tid >> t) & 1u) << ta.out_rank[tp.map[NST - 1].order[t]];
    }
    uint32_t pin[kRegBits], pout[kRegBits];
#pragma unroll
    for (int b = 0; b < kRegBits; ++b) {
        pin[b] = 1u << ta.in_rank[tp.map[0].win[b]];
        pout[b] = 1u << ta.out_rank[tp.map[NST - 1].win[b]];
    }
    // table indices of the per-thread phases exp(i pi z_t / 2^u) (wires of
    // windows >= 1: the earlier wires that are thread bits); tile-independent
    uint32_t pidx[A > 4 ? A : 5];
#pragma unroll
    for (int u = 4; u < A; ++u) pidx[u] = ((tpart[u / 4] & ((1u << u) - 1u)) << (9 - u)) & 1023u;
    const bool twid = !HONLY && (tp.n_et > 0 || tp.n_ef > 0 || tp.y_const != 0);
    constexpr uint32_t amask = (1u << A) - 1u;
    const uint32_t Jt = __brev(tpart[0] & amask) >> (32 - A);
    uint64_t yt = 0;
    for (int e = 0; e < tp.n_et; ++e) yt += (uint64_t)((tpart[0] >> tp.et_bit[e]) & 1u) << tp.et_w[e];

    for (uint64_t j = 0;; ++j) {
        const uint64_t T = tile_of(j);
        if (T >= ntiles) break;
        const int st = (int)(j % kStages);
        double2 *buf = bufs + (size_t)st * (1u << kTmaTileBits);
        mbar_wait(&full[st], (uint32_t)((j / kStages) & 1));
        double2 v[NS];
        {
            uint32_t o[NS];
            o[0] = lin;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] | pin[b];
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = buf[o[k]];
        }
        // twiddle exp(2 pi i Y J / 2^W) of the earlier blocks' R_d gates and
        // the 2^(-A/2) normalisation: J = Jt + sum_b k_b 2^(A-1-b), so the
        // window-bit factors are beta_3, beta_2 = beta_3^2, ...
        if (twid) {
            uint64_t Y = tp.y_const + yt;
            for (int e = 0; e < tp.n_ef; ++e) Y += ((T >> tp.ef_bit[e]) & 1u) << tp.ef_w[e];
            const double2 Ar = root_of_unity(Y * Jt, tp.W, tab, tp.tw);
            const double2 As = make_double2(Ar.x * tp.scale, Ar.y * tp.scale);
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = cmul(v[k], As);
            double2 beta = root_of_unity(Y << (A - 4), tp.W, tab, tp.tw);
#pragma unroll
            for (int b = 3; b >= 0; --b) {
#pragma unroll
                for (int k = 0; k < NS; ++k)
                    if (k & (1 << b)) v[k] = cmul(v[k], beta);
                if (b) beta = cmul(beta, beta);
            }
        } else {
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = make_double2(v[k].x * tp.scale, v[k].y * tp.scale);
        }
#pragma unroll
        for (int s = 0; s < NST; ++s) {
            if (s > 0) {
                uint32_t o[NS];
                o[0] = stp[s - 1];
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                    for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] ^ tp.wswz[s - 1][b];
                __syncthreads();
#pragma unroll
                for (int k = 0; k < NS; ++k) buf[o[k]] = v[k];
                o[0] = stp[s];
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                    for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] ^ tp.wswz[s][b];
                __syncthreads();
#pragma unroll
                for (int k = 0; k < NS; ++k) v[k] = buf[o[k]];
            }
            const int w0 = (4 * s + 4 <= A) ? 4 * s : A - 4;
#pragma unroll
            for (int rb = 0; rb < 4; ++rb) {
                const int u = w0 + rb;
                if (u < 4 * s) continue;   // carried wire (already transformed)
                if (!HONLY) {
                    if (u >= 4) {
                        const double2 P = tab[pidx[u]];
#pragma unroll
                        for (int k = 0; k < NS; ++k)
                            if (k & (1 << rb)) v[k] = cmul(v[k], P);
                    }
#pragma unroll
                    for (int k = 0; k < NS; ++k) {
                        if (!(k & (1 << rb))) continue;
#pragma unroll
                        for (int r2 = 0; r2 < rb; ++r2)
                            if (k & (1 << r2)) v[k] = rot_c<INV>(v[k], rb - r2);
                    }
                }
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    if (k & (1 << rb)) continue;
                    const double2 x = v[k], y = v[k | (1 << rb)];
                    v[k] = make_double2(x.x + y.x, x.y + y.y);
                    v[k | (1 << rb)] = make_double2(x.x - y.x, x.y - y.y);
                }
            }
        }
        {
            uint32_t o[NS];
            o[0] = lout;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] | pout[b];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NS; ++k) buf[o[k]] = v[k];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            int c[5];
            coords(ta.out_first, ta.out_len, T, c);
            tma_store(&out_map, c, buf);
            bulk_wait_read<1>();
            const uint64_t Tn = tile_of(j + kStages - 1);
            if (Tn < ntiles) {
                const int sn = (int)((j + kStages - 1) % kStages);
                coords(ta.in_first, ta.in_len, Tn, c);
                mbar_expect_tx(&full[sn], kTileBytes);
                tma_load(bufs + (size_t)sn * (1u << kTmaTileBits), &in_map, c, &full[sn]);
            }
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Generalised QFT pass (QftGen, qsim_internal.h): the block / window /
// pipeline structure of k_qft_tma, with per-gate data instead of exact roots
// of unity -- noisy H matrices (real 2x2 after their column phase) and noisy
// or missing R_d.  All phases on b_u = 1 before H(u) from outside the pass
// (H's column phase, the R gates of earlier blocks) are one diagonal applied
// at load time: exp(i theta_u), theta_u = hph[u] + the angles of the early
// wires set in this thread (computed once) + those set in the tile id (one
// sincos per wire per tile, shared by the CTA through shared memory).  The
// in-block R gates follow k_qft_tma: a per-thread factor for the thread bits
// and per-slot factors for the window bits, applied once per amplitude.
template <int A>
__global__ void __launch_bounds__(kThreads, 1)
    k_qft_gen(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
              const __grid_constant__ TilePass tp, const __grid_constant__ TmaArgs ta,
              const __grid_constant__ QftGen g, uint64_t ntiles)
{
    static_assert(kRegBits == 4 && kTmaTileBits == 12 && A >= 4 && A <= 10, "window layout");
    constexpr int NST = (A + 3) / 4;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);
    double2 *tileE = bufs + kStages * (1u << kTmaTileBits);   // [2][kGenWires]
    uint64_t *full = reinterpret_cast<uint64_t *>(tileE + 2 * kGenWires);
    const uint32_t tid = threadIdx.x;
    // e^{i (angles of the early wires on fixed bits set in tile T)} for wire tid
    auto tile_phase = [&](uint64_t T, int slot) {
        double th = 0.0;
        for (int e = 0; e < tp.n_ef; ++e)
            if ((T >> tp.ef_bit[e]) & 1u) th += g.phe[tid][tp.ef_w[e]];
        double sn, cs;
        sincos(th, &sn, &cs);
        tileE[slot * kGenWires + tid] = make_double2(cs, sn);
    };
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < A && blockIdx.x < ntiles) tile_phase(blockIdx.x, 0);
    __syncthreads();
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&in_map) : "memory");
        for (uint64_t q = 0; q < kStages - 1; ++q) {
            const uint64_t T = blockIdx.x + q * gridDim.x;
            if (T >= ntiles) break;
            int c[5];
            coords(ta.in_first, ta.in_len, T, c);
            mbar_expect_tx(&full[q], kTileBytes);
            tma_load(bufs + (size_t)q * (1u << kTmaTileBits), &in_map, c, &full[q]);
        }
    }
    constexpr int tb = kTmaTileBits - kRegBits;
    uint32_t tpart[NST], stp[NST];
#pragma unroll
    for (int m = 0; m < NST; ++m) {
        tpart[m] = thread_part(tp.map[m], tb, tid);
        stp[m] = swz(tpart[m]);
    }
    uint32_t lin = 0, lout = 0;
    for (int t = 0; t < tb; ++t) {
        lin |= ((tid >> t) & 1u) << ta.in_rank[tp.map[0].order[t]];
        lout |= ((tid >> t) & 1u) << ta.out_rank[tp.map[NST - 1].order[t]];
    }
    uint32_t pin[kRegBits], pout[kRegBits];
#pragma unroll
    for (int b = 0; b < kRegBits; ++b) {
        pin[b] = 1u << ta.in_rank[tp.map[0].win[b]];
        pout[b] = 1u << ta.out_rank[tp.map[NST - 1].win[b]];
    }
    // per thread: theta_u without the tile part; wires 4.. (thread bits of
    // map 0) summed into one factor, wires 0..3 (map 0's window) kept apart
    double2 thrE[4], athr;
    {
        double thw[A];
#pragma unroll
        for (int u = 0; u < A; ++u) {
            double s = g.hph[u];
            for (int e = 0; e < tp.n_et; ++e)
                if ((tpart[0] >> tp.et_bit[e]) & 1u) s += g.phe[u][tp.et_w[e]];
            for (int i = 0; i < kGenEarly && i < 64; ++i)
                if ((tp.y_const >> i) & 1u) s += g.phe[u][i];
            thw[u] = s;
        }
        double sa = 0.0;
#pragma unroll
        for (int u = 4; u < A; ++u)
            if ((tpart[0] >> u) & 1u) sa += thw[u];
        double sn, cs;
        sincos(sa, &sn, &cs);
        athr = make_double2(cs, sn);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            sincos(thw[u], &sn, &cs);
            thrE[u] = make_double2(cs, sn);
        }
    }
    // per thread: in-block phases of the earlier wires that are thread bits of
    // the wire's own map (windows >= 1)
    double2 pth[A > 4 ? A : 5];
#pragma unroll
    for (int u = 4; u < A; ++u) {
        const int s = u / 4;
        const int w0 = (4 * s + 4 <= A) ? 4 * s : A - 4;
        double2 p = make_double2(1.0, 0.0);
        for (int u2 = 0; u2 < w0; ++u2)
            if ((tpart[s] >> u2) & 1u) p = cmul(p, g.ein[u][u2]);
        pth[u] = p;
    }

    uint64_t j = 0;
    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x, ++j) {
        const int st = (int)(j % kStages);
        double2 *buf = bufs + (size_t)st * (1u << kTmaTileBits);
        // outer phases: slot k gets athr * prod(tile part of thread wires) * prod_{b in k} e_b
        double2 f[NS];
        {
            const double2 *tE = tileE + (j & 1) * kGenWires;
            double2 at = athr;
#pragma unroll
            for (int u = 4; u < A; ++u) {
                const double2 x = tE[u];
                const bool on = (tpart[0] >> u) & 1u;
                at = cmul(at, make_double2(on ? x.x : 1.0, on ? x.y : 0.0));
            }
            f[0] = at;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double2 eb = cmul(thrE[b], tE[b]);
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) f[q | (1 << b)] = cmul(f[q], eb);
            }
        }
        const uint64_t Tn = T + gridDim.x;
        if (tid < A && Tn < ntiles) tile_phase(Tn, (int)((j + 1) & 1));
        mbar_wait(&full[st], (uint32_t)((j / kStages) & 1));
        double2 v[NS];
        {
            uint32_t o[NS];
            o[0] = lin;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] | pin[b];
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = cmul(buf[o[k]], f[k]);
        }
#pragma unroll
        for (int s = 0; s < NST; ++s) {
            if (s > 0) {
                uint32_t o[NS];
                o[0] = stp[s - 1];
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                    for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] ^ tp.wswz[s - 1][b];
                __syncthreads();
#pragma unroll
                for (int k = 0; k < NS; ++k) buf[o[k]] = v[k];
                o[0] = stp[s];
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                    for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] ^ tp.wswz[s][b];
                __syncthreads();
#pragma unroll
                for (int k = 0; k < NS; ++k) v[k] = buf[o[k]];
            }
            const int w0 = (4 * s + 4 <= A) ? 4 * s : A - 4;
#pragma unroll
            for (int rb = 0; rb < 4; ++rb) {
                const int u = w0 + rb;
                if (u < 4 * s) continue;   // carried wire (already transformed)
                // in-block R gates of the earlier wires: factor F[lower window bits]
                if (u >= 4 || rb > 0) {
                    double2 F[1 << 3];
                    F[0] = u >= 4 ? pth[u] : make_double2(1.0, 0.0);
#pragma unroll
                    for (int r2 = 0; r2 < rb; ++r2) {
                        const double2 E = g.ein[u][w0 + r2];
#pragma unroll
                        for (int q = 0; q < (1 << r2); ++q) F[q | (1 << r2)] = cmul(F[q], E);
                    }
#pragma unroll
                    for (int k = 0; k < NS; ++k) {
                        if (!(k & (1 << rb))) continue;
                        const int q = k & ((1 << rb) - 1);
                        if (u < 4 && q == 0) continue;   // factor 1
                        v[k] = cmul(v[k], F[q]);
                    }
                }
                const double h0 = g.Hr[u][0], h1 = g.Hr[u][1], h2 = g.Hr[u][2], h3 = g.Hr[u][3];
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    if (k & (1 << rb)) continue;
                    const double2 x = v[k], y = v[k | (1 << rb)];
                    v[k] = make_double2(fma(h0, x.x, h1 * y.x), fma(h0, x.y, h1 * y.y));
                    v[k | (1 << rb)] = make_double2(fma(h2, x.x, h3 * y.x), fma(h2, x.y, h3 * y.y));
                }
            }
        }
        {
            uint32_t o[NS];
            o[0] = lout;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int q = 0; q < (1 << b); ++q) o[q | (1 << b)] = o[q] | pout[b];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NS; ++k) buf[o[k]] = v[k];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            int c[5];
            coords(ta.out_first, ta.out_len, T, c);
            tma_store(&out_map, c, buf);
            bulk_wait_read<1>();
            const uint64_t Tn2 = T + (uint64_t)(kStages - 1) * gridDim.x;
            if (Tn2 < ntiles) {
                const int sn = (int)((j + kStages - 1) % kStages);
                coords(ta.in_first, ta.in_len, Tn2, c);
                mbar_expect_tx(&full[sn], kTileBytes);
                tma_load(bufs + (size_t)sn * (1u << kTmaTileBits), &in_map, c, &full[sn]);
            }
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Gate-list pass on the TMA pipeline (in place), for passes whose FP64 work
// hides under the transfer: tiles stream in by TMA while the previous tile's
// segments run in registers (ops_common.cuh, transposes in the stage buffer),
// results stream back by TMA store.  One CTA of 128 threads per SM.
__global__ void __launch_bounds__(ops::kOpsThreads, 1)
    k_ops_tma(const __grid_constant__ CUtensorMap map, const __grid_constant__ OpsLaunch L,
              const __grid_constant__ TmaArgs ta, uint64_t ntiles)
{
    using namespace ops;
    static_assert(kTmaTileBits == kTileMaxBits, "tile");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(bufs + kStages * (1u << kTmaTileBits));
    const OpsPass &P = L.P;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map) : "memory");
        for (uint64_t q = 0; q < kStages - 1; ++q) {
            const uint64_t T = blockIdx.x + q * gridDim.x;
            if (T >= ntiles) break;
            int c[5];
            coords(ta.in_first, ta.in_len, T, c);
            mbar_expect_tx(&full[q], kTileBytes);
            tma_load(bufs + (size_t)q * (1u << kTmaTileBits), &map, c, &full[q]);
        }
    }
    const int tb = kTmaTileBits - RB5;
    const OpsSeg &s0 = P.seg[0];
    const OpsSeg &sL = P.seg[P.nseg - 1];
    uint32_t lin = 0, lout = 0;
    for (int t = 0; t < tb; ++t) {
        lin |= ((tid >> t) & 1u) << ta.in_rank[s0.order[t]];
        lout |= ((tid >> t) & 1u) << ta.in_rank[sL.order[t]];
    }
    uint32_t pin[RB5], pout[RB5];
#pragma unroll
    for (int b = 0; b < RB5; ++b) {
        pin[b] = 1u << ta.in_rank[s0.win[b]];
        pout[b] = 1u << ta.in_rank[sL.win[b]];
    }
    uint64_t j = 0;
    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x, ++j) {
        const int st = (int)(j % kStages);
        double2 *buf = bufs + (size_t)st * (1u << kTmaTileBits);
        mbar_wait(&full[st], (uint32_t)((j / kStages) & 1));
        double2 v[NS5];
#pragma unroll
        for (int k = 0; k < NS5; ++k) {
            uint32_t o = lin;
#pragma unroll
            for (int b = 0; b < RB5; ++b)
                if (k & (1 << b)) o |= pin[b];
            v[k] = buf[o];
        }
        run_segments(v, L, T, tid, tb, buf);
        __syncthreads();   // every reader of the stage buffer is done
#pragma unroll
        for (int k = 0; k < NS5; ++k) {
            uint32_t o = lout;
#pragma unroll
            for (int b = 0; b < RB5; ++b)
                if (k & (1 << b)) o |= pout[b];
            buf[o] = v[k];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            int c[5];
            coords(ta.in_first, ta.in_len, T, c);
            tma_store(&map, c, buf);
            bulk_wait_read<1>();
            const uint64_t Tn = T + (uint64_t)(kStages - 1) * gridDim.x;
            if (Tn < ntiles) {
                const int sn = (int)((j + kStages - 1) % kStages);
                coords(ta.in_first, ta.in_len, Tn, c);
                mbar_expect_tx(&full[sn], kTileBytes);
                tma_load(bufs + (size_t)sn * (1u << kTmaTileBits), &map, c, &full[sn]);
            }
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Gate-list pass for FP64-heavy op lists: two 128-thread warpgroups per CTA
// (one CTA per SM) work on alternate tiles (ping-pong) -- eight warps per SM
// doing FP64, as k_ops_pass's two CTAs -- while the tiles arrive by TMA into
// a 3-stage ring: the load of tile j+3 leaves as soon as tile j's last
// transpose has been read, instead of each thread's serialised gather.
// Results go from registers straight to HBM (the stage is free at once).
__global__ void __launch_bounds__(2 * ops::kOpsThreads, 1)
    k_ops_pp(const __grid_constant__ CUtensorMap map, const __grid_constant__ OpsLaunch L,
             const __grid_constant__ TmaArgs ta, double2 *psi, uint64_t ntiles)
{
    using namespace ops;
    static_assert(kTmaTileBits == kTileMaxBits && kStages == 3, "tile / ring");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(bufs + kStages * (1u << kTmaTileBits));
    const OpsPass &P = L.P;
    const uint32_t wg = threadIdx.x / kOpsThreads;
    const uint32_t tid = threadIdx.x % kOpsThreads;
    GOp *ops = reinterpret_cast<GOp *>(full + 8);   // the op list in shared memory (see k_ops_pass)
    {
        const int4 *src = reinterpret_cast<const int4 *>(L.ops);
        int4 *dst = reinterpret_cast<int4 *>(ops);
        const int words = P.nops * (int)(sizeof(GOp) / sizeof(int4));
        for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map) : "memory");
        for (uint64_t q = 0; q < kStages; ++q) {
            const uint64_t T = blockIdx.x + q * gridDim.x;
            if (T >= ntiles) break;
            int c[5];
            coords(ta.in_first, ta.in_len, T, c);
            mbar_expect_tx(&full[q], kTileBytes);
            tma_load(bufs + (size_t)q * (1u << kTmaTileBits), &map, c, &full[q]);
        }
    }
    const int tb = kTmaTileBits - RB5;
    const OpsSeg &s0 = P.seg[0];
    const OpsSeg &sL = P.seg[P.nseg - 1];
    uint32_t lin = 0;
    uint64_t tout = 0;
    for (int t = 0; t < tb; ++t) {
        lin |= ((tid >> t) & 1u) << ta.in_rank[s0.order[t]];
        tout |= (uint64_t)((tid >> t) & 1u) << P.in_pos[sL.order[t]];
    }
    uint32_t pin[RB5];
    uint64_t pout[RB5];
#pragma unroll
    for (int b = 0; b < RB5; ++b) {
        pin[b] = 1u << ta.in_rank[s0.win[b]];
        pout[b] = 1ull << P.in_pos[sL.win[b]];
    }
    const WgSync sync{1u + wg};
    for (uint64_t j = wg;; j += 2) {
        const uint64_t T = blockIdx.x + j * gridDim.x;
        if (T >= ntiles) break;
        const int st = (int)(j % kStages);
        double2 *buf = bufs + (size_t)st * (1u << kTmaTileBits);
        mbar_wait(&full[st], (uint32_t)((j / kStages) & 1));
        double2 v[NS5];
#pragma unroll
        for (int k = 0; k < NS5; ++k) {
            uint32_t o = lin;
#pragma unroll
            for (int b = 0; b < RB5; ++b)
                if (k & (1 << b)) o |= pin[b];
            v[k] = buf[o];
        }
        run_segments(v, L, T, tid, tb, buf, sync, ops);
        // the stage is no longer read: the next load into it may leave
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        sync();
        if (tid == 0) {
            const uint64_t Tn = T + (uint64_t)kStages * gridDim.x;
            if (Tn < ntiles) {
                int c[5];
                coords(ta.in_first, ta.in_len, Tn, c);
                mbar_expect_tx(&full[st], kTileBytes);
                tma_load(buf, &map, c, &full[st]);
            }
        }
        uint64_t ib = 0;
        for (int f = 0; f < P.nfix; ++f) ib |= ((T >> f) & 1u) << P.fin_pos[f];
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
}

// ------------------------------------------------------------------ host
}  // namespace

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
        else
            cudaGetLastError();
    }
    return fn;
}

// Build the 5-D tensor map of one side (in or out).  pos_of_tile[b] = the
// position of tile bit b on this side; fixed position p carries tile-id bit
// fid[p] (-1 for tile positions).  Returns false if the geometry needs more
// than 5 dims or a fixed run is not a consecutive tile-id range.
bool build_side(const double2 *base, int nl, const std::vector<int> &pos_of_tile, const std::vector<int> &fid,
                CUtensorMap &map, int (&first)[5], int (&len)[5], int *rank)
{
    const int tbits = (int)pos_of_tile.size();
    std::vector<int> is_tile(nl, -1);
    for (int b = 0; b < tbits; ++b) is_tile[pos_of_tile[b]] = b;
    // ranks: tile bits ordered by position
    {
        std::vector<int> order(tbits);
        for (int b = 0; b < tbits; ++b) order[b] = b;
        std::sort(order.begin(), order.end(), [&](int x, int y) { return pos_of_tile[x] < pos_of_tile[y]; });
        for (int r = 0; r < tbits; ++r) rank[order[r]] = r;
    }
    if (is_tile[0] < 0) return false;   // the innermost dim must be tile positions
    cuuint64_t gdim[5], gstride[4];
    cuuint32_t box[5], estr[5];
    int nd = 0;
    int p = 0;
    while (p < nl) {
        const bool tilep = is_tile[p] >= 0;
        int q = p;
        if (tilep) {
            while (q < nl && is_tile[q] >= 0 && q - p < (nd == 0 ? 7 : 8)) ++q;
        } else {
            while (q < nl && is_tile[q] < 0 && fid[q] == fid[p] + (q - p)) ++q;
        }
        if (nd == 5) return false;
        const int L = q - p;
        if (nd == 0) {
            gdim[0] = (cuuint64_t)2 << L;   // doubles
            box[0] = 2u << L;
        } else {
            gdim[nd] = (cuuint64_t)1 << L;
            box[nd] = tilep ? (1u << L) : 1u;
            gstride[nd - 1] = (cuuint64_t)16 << p;
        }
        first[nd] = tilep ? 0 : fid[p];
        len[nd] = tilep ? 0 : L;
        ++nd;
        p = q;
    }
    while (nd < 5) {
        gdim[nd] = 1;
        box[nd] = 1;
        gstride[nd - 1] = (cuuint64_t)16 << nl;   // size-1 padding dims: any 16-B multiple
        first[nd] = 0;
        len[nd] = 0;
        ++nd;
    }
    for (int d = 0; d < 5; ++d) estr[d] = 1;
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    // L2 promotion no wider than the box's contiguous run (a 256-byte
    // promotion of 128-byte runs also fetches the neighbouring run)
    const uint32_t run_bytes = box[0] * 8u;
    CUtensorMapL2promotion prom = run_bytes >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                  : run_bytes >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                     : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    static const int prom_env = getenv("QSIM_L2PROM") ? atoi(getenv("QSIM_L2PROM")) : -1;   // measurement knob
    if (prom_env >= 0)
        prom = prom_env >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
               : prom_env >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
               : prom_env >= 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void *)base, gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

namespace {

template <int NM>
void launch_tma_nm(Handle *h, const CUtensorMap &im, const CUtensorMap &om, const TilePass &tp, const TmaArgs &ta)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const size_t smem = (size_t)kStages * kTileBytes + 1024 * sizeof(double2) + kStages * sizeof(uint64_t);
    static uint64_t attr = 0;
    if (first_use_on_device(attr)) {
        cudaFuncSetAttribute(k_tile_tma<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    const uint64_t ntiles = 1ull << tp.nfix;
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)h->num_sms);
    prof_begin(h);
    k_tile_tma<NM><<<grid, kThreads, smem, h->stream>>>(im, om, tp, ta, ntiles);
    prof_end(h, "k_tile_tma", (1ull << (tp.tbits + tp.nfix)) * 32);
}

template <int A, bool INV, bool HONLY>
void launch_fixed(Handle *h, const CUtensorMap &im, const CUtensorMap &om, const TilePass &tp, const TmaArgs &ta)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const size_t smem = (size_t)kStages * kTileBytes + 1024 * sizeof(double2) + kStages * sizeof(uint64_t);
    static uint64_t attr = 0;
    if (first_use_on_device(attr)) {
        cudaFuncSetAttribute(k_qft_tma<A, INV, HONLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    const uint64_t ntiles = 1ull << tp.nfix;
    // tiles per CTA group (QSIM_TILE_GROUP: measurement knob); groups keep the grid size
    static const int genv = getenv("QSIM_TILE_GROUP") ? atoi(getenv("QSIM_TILE_GROUP")) : 0;
    int gbits = genv;
    while (gbits > 0 && (ntiles >> gbits) < (uint64_t)h->num_sms) --gbits;
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles >> gbits, (uint64_t)h->num_sms);
    prof_begin(h);
    k_qft_tma<A, INV, HONLY><<<grid, kThreads, smem, h->stream>>>(im, om, tp, ta, ntiles, gbits);
    prof_end(h, "k_qft_tma", (1ull << (tp.tbits + tp.nfix)) * 32);
}

template <int A>
bool launch_fixed_a(Handle *h, const CUtensorMap &im, const CUtensorMap &om, const TilePass &tp, const TmaArgs &ta)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    if (tp.hadamard_only) launch_fixed<A, false, true>(h, im, om, tp, ta);
    else if (tp.inverse) launch_fixed<A, true, false>(h, im, om, tp, ta);
    else launch_fixed<A, false, false>(h, im, om, tp, ta);
    return true;
}

}  // namespace

// Try the TMA path for a planned pass (tp as given to launch_tile_pass).
// Returns false (nothing launched) when the geometry does not fit.
bool launch_tile_pass_tma(Handle *h, const TilePass &tp_in, const double2 *in, double2 *out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    if (tp_in.tbits != kTmaTileBits || getenv("QSIM_NO_TMA")) return false;
    TilePass tp = tp_in;
    finish_tile_pass(tp);
    std::vector<int> fid_in(h->nl, -1), fid_out(h->nl, -1);
    for (int f = 0; f < tp.nfix; ++f) {
        fid_in[tp.fin_pos[f]] = f;
        fid_out[tp.fout_pos[f]] = f;
    }
    std::vector<int> tin(tp.in_pos, tp.in_pos + tp.tbits), tout(tp.out_pos, tp.out_pos + tp.tbits);
    CUtensorMap im, om;
    TmaArgs ta;
    std::memset(&ta, 0, sizeof ta);
    if (!build_side(in, h->nl, tin, fid_in, im, ta.in_first, ta.in_len, ta.in_rank)) return false;
    if (!build_side(out, h->nl, tout, fid_out, om, ta.out_first, ta.out_len, ta.out_rank)) return false;
    // specialised kernel: 4..10 active wires, windows as planned, early tile
    // bits outside window 0
    const int nst = (tp.a + 3) / 4;
    if (!getenv("QSIM_NO_FIXED") && tp.a >= 4 && tp.a <= 10 && tp.nmaps == nst && tp.twiddle_fast) {
        switch (tp.a) {
        case 4: return launch_fixed_a<4>(h, im, om, tp, ta);
        case 5: return launch_fixed_a<5>(h, im, om, tp, ta);
        case 6: return launch_fixed_a<6>(h, im, om, tp, ta);
        case 7: return launch_fixed_a<7>(h, im, om, tp, ta);
        case 8: return launch_fixed_a<8>(h, im, om, tp, ta);
        case 9: return launch_fixed_a<9>(h, im, om, tp, ta);
        default: return launch_fixed_a<10>(h, im, om, tp, ta);
        }
    }
    switch (tp.nmaps) {
    case 1: launch_tma_nm<1>(h, im, om, tp, ta); break;
    case 2: launch_tma_nm<2>(h, im, om, tp, ta); break;
    case 3: launch_tma_nm<3>(h, im, om, tp, ta); break;
    case 4: launch_tma_nm<4>(h, im, om, tp, ta); break;
    case 5: launch_tma_nm<5>(h, im, om, tp, ta); break;
    default: launch_tma_nm<6>(h, im, om, tp, ta); break;
    }
    return true;
}

template <int A>
void launch_gen_a(Handle *h, const CUtensorMap &im, const CUtensorMap &om, const TilePass &tp, const TmaArgs &ta,
                  const QftGen &g)
{
    const size_t smem = (size_t)kStages * kTileBytes + 2 * kGenWires * sizeof(double2) + kStages * sizeof(uint64_t);
    static uint64_t attr = 0;
    if (first_use_on_device(attr))
        cudaFuncSetAttribute(k_qft_gen<A>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint64_t ntiles = 1ull << tp.nfix;
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)h->num_sms);
    prof_begin(h);
    k_qft_gen<A><<<grid, kThreads, smem, h->stream>>>(im, om, tp, ta, g, ntiles);
    prof_end(h, "k_qft_gen", (1ull << (tp.tbits + tp.nfix)) * 32);
}

// geometry of a generalised pass: tensor maps and the specialised window layout
static bool gen_geometry(Handle *h, const TilePass &tp_in, const double2 *in, double2 *out, TilePass &tp,
                         CUtensorMap &im, CUtensorMap &om, TmaArgs &ta)
{
    if (tp_in.tbits != kTmaTileBits || getenv("QSIM_NO_TMA")) return false;
    tp = tp_in;
    finish_tile_pass(tp);
    const int nst = (tp.a + 3) / 4;
    if (tp.a < 4 || tp.a > kGenWires || tp.nmaps != nst || !tp.twiddle_fast) return false;
    for (int e = 0; e < tp.n_et; ++e) if (tp.et_w[e] >= kGenEarly) return false;
    for (int e = 0; e < tp.n_ef; ++e) if (tp.ef_w[e] >= kGenEarly) return false;
    if (tp.y_const >> kGenEarly) return false;
    std::vector<int> fid_in(h->nl, -1), fid_out(h->nl, -1);
    for (int f = 0; f < tp.nfix; ++f) {
        fid_in[tp.fin_pos[f]] = f;
        fid_out[tp.fout_pos[f]] = f;
    }
    std::vector<int> tin(tp.in_pos, tp.in_pos + tp.tbits), tout(tp.out_pos, tp.out_pos + tp.tbits);
    std::memset(&ta, 0, sizeof ta);
    if (!build_side(in, h->nl, tin, fid_in, im, ta.in_first, ta.in_len, ta.in_rank)) return false;
    if (!build_side(out, h->nl, tout, fid_out, om, ta.out_first, ta.out_len, ta.out_rank)) return false;
    return true;
}

bool qft_gen_feasible(Handle *h, const TilePass &tp_in)
{
    TilePass tp;
    CUtensorMap im, om;
    TmaArgs ta;
    return gen_geometry(h, tp_in, h->psi, h->psi, tp, im, om, ta);
}

bool launch_qft_gen_tma(Handle *h, const TilePass &tp_in, const QftGen &g, const double2 *in, double2 *out)
{
    cudaSetDevice(h->device);
    TilePass tp;
    CUtensorMap im, om;
    TmaArgs ta;
    if (!gen_geometry(h, tp_in, in, out, tp, im, om, ta)) return false;
    switch (tp.a) {
    case 4: launch_gen_a<4>(h, im, om, tp, ta, g); break;
    case 5: launch_gen_a<5>(h, im, om, tp, ta, g); break;
    case 6: launch_gen_a<6>(h, im, om, tp, ta, g); break;
    case 7: launch_gen_a<7>(h, im, om, tp, ta, g); break;
    case 8: launch_gen_a<8>(h, im, om, tp, ta, g); break;
    case 9: launch_gen_a<9>(h, im, om, tp, ta, g); break;
    default: launch_gen_a<10>(h, im, om, tp, ta, g); break;
    }
    return true;
}

bool launch_ops_pass_tma(Handle *h, const OpsLaunch &L)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const OpsPass &P = L.P;
    if (P.tbits != kTmaTileBits || getenv("QSIM_NO_TMA")) return false;
    std::vector<int> fid(h->nl, -1);
    for (int f = 0; f < P.nfix; ++f) fid[P.fin_pos[f]] = f;
    std::vector<int> tp(P.in_pos, P.in_pos + P.tbits);
    CUtensorMap im;
    TmaArgs ta;
    std::memset(&ta, 0, sizeof ta);
    if (!build_side(h->psi, h->nl, tp, fid, im, ta.in_first, ta.in_len, ta.in_rank)) return false;
    const size_t smem = (size_t)kStages * kTileBytes + 8 * sizeof(uint64_t);
    static uint64_t attr = 0;
    if (first_use_on_device(attr)) {
        cudaFuncSetAttribute(k_ops_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    const uint64_t ntiles = 1ull << P.nfix;
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)h->num_sms);
    prof_begin(h);
    k_ops_tma<<<grid, ops::kOpsThreads, smem, h->stream>>>(im, L, ta, ntiles);
    prof_end(h, "k_ops_tma", (1ull << (P.tbits + P.nfix)) * 32);
    return true;
}

}  // namespace qs

namespace qs {

// FP64-heavy gate-list pass through k_ops_pp; false = the tile is not a <= 5-D box
bool launch_ops_pass_pp(Handle *h, const OpsLaunch &L)
{
    cudaSetDevice(h->device);
    const OpsPass &P = L.P;
    static const bool off = getenv("QSIM_NO_OPS_PP") != nullptr;
    if (P.tbits != kTmaTileBits || off || getenv("QSIM_NO_TMA")) return false;
    std::vector<int> fid(h->nl, -1);
    for (int f = 0; f < P.nfix; ++f) fid[P.fin_pos[f]] = f;
    std::vector<int> tp(P.in_pos, P.in_pos + P.tbits);
    CUtensorMap im;
    TmaArgs ta;
    std::memset(&ta, 0, sizeof ta);
    if (!build_side(h->psi, h->nl, tp, fid, im, ta.in_first, ta.in_len, ta.in_rank)) return false;
    const size_t smem = (size_t)kStages * kTileBytes + 8 * sizeof(uint64_t) + (size_t)P.nops * sizeof(GOp);
    static uint64_t attr = 0;
    if (first_use_on_device(attr))
        cudaFuncSetAttribute(k_ops_pp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((size_t)kStages * kTileBytes + 8 * sizeof(uint64_t) + kOpsParam * sizeof(GOp)));
    const uint64_t ntiles = 1ull << P.nfix;
    const unsigned grid = (unsigned)std::min<uint64_t>((ntiles + 1) / 2, (uint64_t)h->num_sms);
    prof_begin(h);
    k_ops_pp<<<grid, 2 * ops::kOpsThreads, smem, h->stream>>>(im, L, ta, h->psi, ntiles);
    prof_end(h, "k_ops_pp", (1ull << (P.tbits + P.nfix)) * 32);
    return true;
}

}  // namespace qs
