// k_qft13.cu -- fused QFT / H pass on 2^13-amplitude tiles (sm_100a).
//
// Same block arithmetic as k_tma.cu's k_qft_tma (§2.3.2:
// the R_{k-j} of earlier blocks as one Cooley-Tukey twiddle, the R_d inside
// the block as phases before each H, H unnormalised with 2^(-a/2) folded into
// the twiddle), on a tile twice as large so that a pass carries one more
// passive low position: a 9-wire pass reads and writes 256-byte runs (4
// passive bits) and a 10-wire pass 128-byte runs, which is what lets the
// n = 28 QFT run in three HBM passes (10, 9, 9 wires) instead of four.
// Measured on this B200 (tools/pass_pattern.cu, profiles/): a pass streams at
// ~4.5 TB/s with 64-byte read runs, ~5.7 with 128, >= 6.1 with >= 256.
//
// Data path, one CTA (8 warps, 32 amplitudes per thread) per SM:
//   * a tile lands by TMA as four 32 KiB quarter boxes in a ring of seven
//     quarter slots (mbarrier per slot); the next tile's first three quarters
//     are in flight while a tile is computed, its fourth (and the tile after
//     next's first three) leave as soon as this tile's transpose has been
//     read, so 96-128 KiB of loads are in flight per SM;
//   * registers hold the tile in two 5-bit windows: window 0 = wires 0..4,
//     window 1 = wires a-5..a-1; one XOR-swizzled shared-memory transpose
//     (in the tile's own four slots) between them;
//   * results go from registers straight to HBM (the last window's thread
//     bits are ordered by output position, so a warp stores 512-byte runs
//     when the output is contiguous).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mbar.cuh"
#include "qsim_internal.h"
#include "tile_common.cuh"
#include "tma_host.h"

namespace qs {

namespace {

constexpr int kTB = 13;                    // tile bits
constexpr int kQB = 11;                    // quarter-slot bits
constexpr int kSlots = 7;
constexpr uint32_t kSlotAmps = 1u << kQB;
constexpr uint32_t kSlotBytes = 16u << kQB;
constexpr int kWB = 5;                     // register window bits
constexpr int kNS = 1 << kWB;              // amplitudes per thread
constexpr int kThr = 1 << (kTB - kWB);     // 256 threads
constexpr int kThrBits = kTB - kWB;        // 8

struct Q13 {
    int a, W;
    double scale, tw;
    int order0[kThrBits], order1[kThrBits];   // thread bit t -> tile bit (map 0 / map 1)
    int in_rank[kTB];                         // landing index bit of tile bit b (rank of its input position)
    int out_pos[kTB];                         // output local position of tile bit b
    int nfix;
    // tile-id bit runs: bits [src, src+len) of T go to bits [dst, dst+len) of
    // the output address (o*) / of the early-wire value Y (e*)
    int n_orun, orun_src[kMaxFixedBits], orun_len[kMaxFixedBits], orun_dst[kMaxFixedBits];
    int n_erun, erun_src[kMaxFixedBits], erun_len[kMaxFixedBits], erun_dst[kMaxFixedBits];
    int n_et, et_bit[kTB], et_w[kTB];         // early wires on tile bits
    int n_ef;                                 // early wires on tile-id bits (as erun)
    uint64_t y_const;
    int qe0, qe1;                             // ext-id bits of the quarter index (landing ranks 11, 12; -1: global)
    int pb;                                   // window-1 bit whose output position is 0 (-1: none): 32-byte stores
    int in_first[5], in_len[5];               // tensor-map dim -> ext-id bit run
    // rank-group pass (the exchange fused into the pass, peer memory): ng
    // tile bits sit on rank bits -- the highest-ranked tile bits, i.e. the
    // quarter bits -- so the tile's rows live in 2^ng shards; quarter q comes
    // from shard (q >> (2 - ng)) through its own tensor map, every element is
    // stored into the shard its global bits name, and this rank takes the
    // tiles whose split bits equal its own rank bits
    int ng;
    int split_bit[2];                         // tile-id bits fixed per rank (ascending)
    uint64_t split_val;
    int gthr[2], gwin[2];                     // map-1 thread bit / window bit of global tile bit i (-1: not)
    double2 *outb[4];                         // shard of global-bit combination c
};

__device__ __forceinline__ void tma_load5(void *dst, const CUtensorMap *map, const int (&c)[5], uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(bar))
        : "memory");
}

// insert bit value v at position e of x
__device__ __forceinline__ uint64_t ins_bit(uint64_t x, int e, uint64_t v)
{
    const uint64_t lo = x & ((1ull << e) - 1);
    return ((x >> e) << (e + 1)) | (v << e) | lo;
}

// two adjacent amplitudes in one 256-bit streaming store (STG.E.ENL2.256)
__device__ __forceinline__ void st_pair_cs(double2 *p, double2 a, double2 b)
{
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                 : "memory");
}

// window-1 register slots k and k | 2^PB hold neighbouring output amplitudes
// (window bit PB sits on output position 0): 16 stores of 32 bytes per thread
template <int PB>
__device__ __forceinline__ void store_pairs(double2 *__restrict__ out, uint64_t ib, const uint64_t (&pout)[5],
                                            const double2 (&v)[32])
{
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if (k & (1 << PB)) continue;
        uint64_t o = ib;
#pragma unroll
        for (int b = 0; b < 5; ++b)
            if (k & (1 << b)) o |= pout[b];
        st_pair_cs(out + o, v[k], v[k | (1 << PB)]);
    }
}

// 13-bit XOR swizzle (16-byte granules; linear over GF(2))
__device__ __forceinline__ uint32_t swz13(uint32_t ti)
{
    const uint32_t f = (ti >> 3) ^ (ti >> 6) ^ (ti >> 9) ^ (ti >> 12);
    return ti ^ (f & 7u);
}

// exp(i pi j / 16), j = 0..31 (compile-time index in the unrolled loops)
__device__ constexpr double kC32[32] = {
    1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708, 0.70710678118654752440,
    0.55557023301960222474, 0.38268343236508977173, 0.19509032201612826785, 0.0, -0.19509032201612826785,
    -0.38268343236508977173, -0.55557023301960222474, -0.70710678118654752440, -0.83146961230254523708,
    -0.92387953251128675613, -0.98078528040323044913, -1.0, -0.98078528040323044913, -0.92387953251128675613,
    -0.83146961230254523708, -0.70710678118654752440, -0.55557023301960222474, -0.38268343236508977173,
    -0.19509032201612826785, 0.0, 0.19509032201612826785, 0.38268343236508977173, 0.55557023301960222474,
    0.70710678118654752440, 0.83146961230254523708, 0.92387953251128675613, 0.98078528040323044913};

// c * exp(+-i pi j / 16) for a compile-time j (quarter turns are free)
template <bool INV>
__device__ __forceinline__ double2 rot16(double2 c, int j)
{
    j &= 31;
    if (j == 0) return c;
    if (j == 8) return INV ? make_double2(c.y, -c.x) : make_double2(-c.y, c.x);
    if (j == 16) return make_double2(-c.x, -c.y);
    if (j == 24) return INV ? make_double2(-c.y, c.x) : make_double2(c.y, -c.x);
    const double co = kC32[j], si = INV ? -kC32[(j + 24) & 31] : kC32[(j + 24) & 31];   // sin = cos(x - pi/2)
    return make_double2(fma(c.x, co, -c.y * si), fma(c.x, si, c.y * co));
}

// exp(+-2 pi i m / 1024) from two 32-entry shared-memory tables (the seven
// 32 KiB slots leave ~3 KB): coarse[m >> 5] * fine[m & 31]
__device__ __forceinline__ double2 root1024(uint32_t m, const double2 *coarse, const double2 *fine)
{
    return tile::cmul(coarse[(m >> 5) & 31u], fine[m & 31u]);
}

// exp(+-2 pi i t / 2^W) (tw = +-2 pi / 2^W): the 10 leading bits from the
// tables, a Taylor series for the remainder angle (|theta| < 2 pi / 1024)
__device__ __forceinline__ double2 root13(uint64_t t, int W, const double2 *coarse, const double2 *fine, double tw)
{
    if (W <= 10) return root1024((uint32_t)(t << (10 - W)) & 1023u, coarse, fine);
    const uint64_t hi = t >> (W - 10);
    const uint64_t lo = t & ((1ull << (W - 10)) - 1);
    double2 p = root1024((uint32_t)hi & 1023u, coarse, fine);
    if (lo) {
        const double th = (double)lo * tw;
        const double t2 = th * th;
        const double c = fma(fma(fma(-t2, 1.0 / 720.0, 1.0 / 24.0), t2, -0.5), t2, 1.0);
        const double sn = th * fma(fma(fma(-t2, 1.0 / 5040.0, 1.0 / 120.0), t2, -1.0 / 6.0), t2, 1.0);
        p = tile::cmul(p, make_double2(c, sn));
    }
    return p;
}

template <int A, bool INV, bool HONLY>
__global__ void __launch_bounds__(kThr, 1)
    k_qft13(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap in_map1,
            const __grid_constant__ CUtensorMap in_map2, const __grid_constant__ CUtensorMap in_map3,
            double2 *__restrict__ out, const __grid_constant__ Q13 P, uint64_t ntiles)
{
    static_assert(A >= kWB && A <= 10, "two 5-bit windows");
    constexpr int W1 = A - kWB;               // first wire of window 1
    constexpr double SG = INV ? -1.0 : 1.0;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double2 *slots = reinterpret_cast<double2 *>(smem_raw);
    double2 *coarse = slots + kSlots * kSlotAmps;   // exp(+-2 pi i k / 32)
    double2 *fine = coarse + 32;                     // exp(+-2 pi i k / 1024), k < 32
    uint64_t *bar = reinterpret_cast<uint64_t *>(fine + 32);
    const uint32_t tid = threadIdx.x;

    if (tid == 0) {
        for (int s = 0; s < kSlots; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (!HONLY && tid < 64) {
        double sn, cs;
        sincospi((double)(tid & 31) / (tid < 32 ? 16.0 : 512.0), &sn, &cs);
        (tid < 32 ? coarse : fine)[tid & 31] = make_double2(cs, SG * sn);
    }
    __syncthreads();

    // quarter load s (s = 4 j + q: tile j of this CTA, quarter q) into slot s % 7
    // this rank's t-th tile -> the full tile id (the split bits carry the rank's bits)
    auto full_tile = [&](uint64_t t) -> uint64_t {
        for (int i = 0; i < P.ng; ++i) t = ins_bit(t, P.split_bit[i], (P.split_val >> i) & 1);
        return t;
    };
    auto issue = [&](uint64_t s) {
        const uint64_t t = blockIdx.x + (s >> 2) * (uint64_t)gridDim.x;
        if (t >= ntiles) return;
        const uint64_t T = full_tile(t);
        const uint64_t q = s & 3;
        uint64_t X = T;
        if (P.qe0 >= 0) X = ins_bit(X, P.qe0, q & 1);
        if (P.qe1 >= 0) X = ins_bit(X, P.qe1, q >> 1);
        int c[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) c[d] = P.in_len[d] ? (int)((X >> P.in_first[d]) & ((1ull << P.in_len[d]) - 1)) : 0;
        const int sl = (int)(s % kSlots);
        mbar_expect_tx(&bar[sl], kSlotBytes);
        const int m = P.ng == 0 ? 0 : (int)(q >> (2 - P.ng));
        const CUtensorMap *mp = m == 0 ? &in_map : m == 1 ? &in_map1 : m == 2 ? &in_map2 : &in_map3;
        tma_load5(slots + (size_t)sl * kSlotAmps, mp, c, &bar[sl]);
    };
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&in_map) : "memory");
        for (uint64_t s = 0; s < kSlots; ++s) issue(s);
    }

    // ---- per-thread constants
    uint32_t tp0 = 0, tp1 = 0, lin = 0;
    uint64_t tout = 0;
#pragma unroll
    for (int t = 0; t < kThrBits; ++t) {
        const uint32_t bit = (tid >> t) & 1u;
        tp0 |= bit << P.order0[t];
        tp1 |= bit << P.order1[t];
        lin |= bit << P.in_rank[P.order0[t]];
        if (P.out_pos[P.order1[t]] >= 0) tout |= (uint64_t)bit << P.out_pos[P.order1[t]];
    }
    uint32_t pin[kWB];
    uint64_t pout[kWB];
#pragma unroll
    for (int b = 0; b < kWB; ++b) {
        pin[b] = 1u << P.in_rank[b];
        pout[b] = P.out_pos[W1 + b] >= 0 ? 1ull << P.out_pos[W1 + b] : 0ull;   // -1: a global bit
    }
    // global-bit combination of this thread's part of its elements (map 1)
    uint32_t gtid = 0;
    for (int i = 0; i < P.ng; ++i)
        if (P.gthr[i] >= 0) gtid |= ((tid >> P.gthr[i]) & 1u) << i;
    const uint32_t stp0 = swz13(tp0), stp1 = swz13(tp1);
    // J of the thread bits of map 0 (the window-0 bits are wires 0..4: weights 2^(A-1-b))
    constexpr uint32_t amask = (1u << A) - 1u;
    const uint32_t Jt = __brev(tp0 & amask) >> (32 - A);
    uint64_t yt = 0;
    for (int e = 0; e < P.n_et; ++e) yt += (uint64_t)((tp0 >> P.et_bit[e]) & 1u) << P.et_w[e];
    const bool twid = !HONLY && (P.n_et > 0 || P.n_ef > 0 || P.y_const != 0);
    // window-1 wires: phases exp(i pi sum_{u' < u, thread bits} y_u' 2^(u'-u)) from the table
    uint32_t pidx[kWB];
#pragma unroll
    for (int b = 0; b < kWB; ++b) {
        const int u = W1 + b;
        pidx[b] = ((tp1 & ((1u << u) - 1u)) << (9 - u)) & 1023u;
    }

    for (uint64_t j = 0;; ++j) {
        const uint64_t tt = blockIdx.x + j * (uint64_t)gridDim.x;
        if (tt >= ntiles) break;
        const uint64_t T = full_tile(tt);
        const uint32_t s0 = (uint32_t)((4 * j) % kSlots);   // slot of quarter 0; quarter q in (s0 + q) % 7
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t s = 4 * j + q;
            mbar_wait(&bar[s % kSlots], (uint32_t)((s / kSlots) & 1));
        }
        auto slot_base = [&](uint32_t q) -> uint32_t {
            uint32_t sl = s0 + q;
            if (sl >= kSlots) sl -= kSlots;
            return sl * kSlotAmps;
        };
        double2 v[kNS];
#pragma unroll
        for (int k = 0; k < kNS; ++k) {
            uint32_t r = lin;
#pragma unroll
            for (int b = 0; b < kWB; ++b)
                if (k & (1 << b)) r |= pin[b];
            v[k] = slots[slot_base(r >> kQB) + (r & (kSlotAmps - 1))];
        }
        // ---- twiddle exp(2 pi i Y J / 2^W) and the 2^(-A/2) normalisation
        if (twid) {
            uint64_t Y = P.y_const + yt;
            for (int e = 0; e < P.n_erun; ++e)
                Y += ((T >> P.erun_src[e]) & ((1ull << P.erun_len[e]) - 1)) << P.erun_dst[e];
            const double2 Ar = root13(Y * Jt, P.W, coarse, fine, P.tw);
            const double2 As = make_double2(Ar.x * P.scale, Ar.y * P.scale);
            // slot factor As * prod_b beta_b^{k_b}, beta_b = root(Y 2^(A-1-b)), walked
            // in Gray-code order: one complex multiply per slot to update it
            double2 beta[kWB];
            beta[kWB - 1] = root13(Y << (A - kWB), P.W, coarse, fine, P.tw);
#pragma unroll
            for (int b = kWB - 2; b >= 0; --b) beta[b] = tile::cmul(beta[b + 1], beta[b + 1]);
            double2 f = As;
            v[0] = tile::cmul(v[0], f);
#pragma unroll
            for (int i = 1; i < kNS; ++i) {
                const int g = i ^ (i >> 1), gp = (i - 1) ^ ((i - 1) >> 1);
                const int b = (g ^ gp) == 1 ? 0 : (g ^ gp) == 2 ? 1 : (g ^ gp) == 4 ? 2 : (g ^ gp) == 8 ? 3 : 4;
                f = (g >> b) & 1 ? tile::cmul(f, beta[b]) : tile::cmul(f, make_double2(beta[b].x, -beta[b].y));
                v[g] = tile::cmul(v[g], f);
            }
        } else {
#pragma unroll
            for (int k = 0; k < kNS; ++k) v[k] = make_double2(v[k].x * P.scale, v[k].y * P.scale);
        }
        // ---- window 0: wires 0..4 (no earlier wires of this block outside the window)
#pragma unroll
        for (int rb = 0; rb < kWB; ++rb) {
            if (!HONLY && rb > 0) {
#pragma unroll
                for (int k = 0; k < kNS; ++k) {
                    if (!(k & (1 << rb))) continue;
                    // exp(i pi sum_{r2 < rb} k_r2 2^(r2 - rb)) = exp(i pi (k mod 2^rb) / 2^rb)
                    v[k] = rot16<INV>(v[k], (k & ((1 << rb) - 1)) << (4 - rb));
                }
            }
#pragma unroll
            for (int k = 0; k < kNS; ++k) {
                if (k & (1 << rb)) continue;
                const double2 x = v[k], y = v[k | (1 << rb)];
                v[k] = make_double2(x.x + y.x, x.y + y.y);
                v[k | (1 << rb)] = make_double2(x.x - y.x, x.y - y.y);
            }
        }
        // ---- transpose to window 1 through the tile's own slots (swizzled, tile-bit index)
        __syncthreads();   // every landing read of this tile is done
#pragma unroll
        for (int k = 0; k < kNS; ++k) {
            uint32_t ti = stp0;
#pragma unroll
            for (int b = 0; b < kWB; ++b)
                if (k & (1 << b)) ti ^= swz13(1u << b);
            slots[slot_base(ti >> kQB) + (ti & (kSlotAmps - 1))] = v[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kNS; ++k) {
            uint32_t ti = stp1;
#pragma unroll
            for (int b = 0; b < kWB; ++b)
                if (k & (1 << b)) ti ^= swz13(1u << (W1 + b));
            v[k] = slots[slot_base(ti >> kQB) + (ti & (kSlotAmps - 1))];
        }
        // the tile's slots are free: the next loads may overwrite them
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0)
            for (uint64_t s = 4 * j + kSlots; s < 4 * j + kSlots + 4; ++s) issue(s);
        // ---- window 1: wires W1..A-1 (wires < kWB were transformed in window 0)
#pragma unroll
        for (int rb = 0; rb < kWB; ++rb) {
            const int u = W1 + rb;
            if (u < kWB) continue;
            if (!HONLY) {
                const double2 Pt = root1024(pidx[rb], coarse, fine);
#pragma unroll
                for (int k = 0; k < kNS; ++k) {
                    if (!(k & (1 << rb))) continue;
                    // earlier wires of the window (slot bits r2 < rb): exp(i pi (k mod 2^rb) / 2^rb)
                    v[k] = rot16<INV>(tile::cmul(v[k], Pt), (k & ((1 << rb) - 1)) << (4 - rb));
                }
            }
#pragma unroll
            for (int k = 0; k < kNS; ++k) {
                if (k & (1 << rb)) continue;
                const double2 x = v[k], y = v[k | (1 << rb)];
                v[k] = make_double2(x.x + y.x, x.y + y.y);
                v[k | (1 << rb)] = make_double2(x.x - y.x, x.y - y.y);
            }
        }
        // ---- store from registers
        uint64_t ib = tout;
        for (int e = 0; e < P.n_orun; ++e)
            ib |= ((T >> P.orun_src[e]) & ((1ull << P.orun_len[e]) - 1)) << P.orun_dst[e];
        if (P.ng == 0 && P.pb >= 0) {
            switch (P.pb) {
            case 0: store_pairs<0>(out, ib, pout, v); break;
            case 1: store_pairs<1>(out, ib, pout, v); break;
            case 2: store_pairs<2>(out, ib, pout, v); break;
            case 3: store_pairs<3>(out, ib, pout, v); break;
            default: store_pairs<4>(out, ib, pout, v); break;
            }
        } else if (P.ng == 0) {
#pragma unroll
            for (int k = 0; k < kNS; ++k) {
                uint64_t o = ib;
#pragma unroll
                for (int b = 0; b < kWB; ++b)
                    if (k & (1 << b)) o |= pout[b];
                __stcs(out + o, v[k]);
            }
        } else {
            // rank-group pass: each element goes to the shard its global bits name
#pragma unroll
            for (int k = 0; k < kNS; ++k) {
                uint64_t o = ib;
#pragma unroll
                for (int b = 0; b < kWB; ++b)
                    if (k & (1 << b)) o |= pout[b];
                uint32_t g = gtid;
                for (int i = 0; i < P.ng; ++i)
                    if (P.gwin[i] >= 0) g |= (uint32_t)((k >> P.gwin[i]) & 1) << i;
                __stcs(P.outb[g] + o, v[k]);
            }
        }
    }
}

template <int A, bool INV, bool HONLY>
void launch13(Handle *h, const CUtensorMap (&im)[4], double2 *out, const Q13 &P, uint64_t ntiles)
{
    const size_t smem = (size_t)kSlots * kSlotBytes + 64 * sizeof(double2) + kSlots * sizeof(uint64_t);
    static uint64_t attr = 0;
    if (first_use_on_device(attr))
        cudaFuncSetAttribute(k_qft13<A, INV, HONLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)h->num_sms);
    prof_begin(h);
    k_qft13<A, INV, HONLY><<<grid, kThr, smem, h->stream>>>(im[0], im[1], im[2], im[3], out, P, ntiles);
    prof_end(h, "k_qft13", (ntiles << kTB) * 32);
}

template <int A>
void launch13_a(Handle *h, const CUtensorMap (&im)[4], double2 *out, const Q13 &P, uint64_t ntiles, bool inv,
                bool honly)
{
    if (honly) launch13<A, false, true>(h, im, out, P, ntiles);
    else if (inv) launch13<A, true, false>(h, im, out, P, ntiles);
    else launch13<A, false, false>(h, im, out, P, ntiles);
}

}  // namespace

bool launch_qft13(Handle *h, const Qft13Desc &d, const double2 *in, double2 *out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    if (d.a < kWB || d.a > 10 || h->nl < kTB + 2 || getenv("QSIM_NO_TMA")) return false;
    // test hook: decline the k-th 13-bit pass of the process (exercises the
    // callers' fall-back paths, e.g. a free-layout plan that fails part-way)
    static const int fail_at = getenv("QSIM_TEST_Q13_DECLINE") ? atoi(getenv("QSIM_TEST_Q13_DECLINE")) : -1;
    static int calls = 0;
    if (fail_at >= 0 && calls++ == fail_at) return false;
    Q13 P;
    std::memset(&P, 0, sizeof P);
    P.a = d.a;
    P.W = d.W;
    P.scale = d.scale;
    P.tw = (d.inverse ? -1.0 : 1.0) * 6.283185307179586476925286766559 / std::ldexp(1.0, d.W);
    const int nl = h->nl;
    // landing ranks: tile bits ordered by input position
    std::vector<int> byin(kTB);
    for (int b = 0; b < kTB; ++b) byin[b] = b;
    std::sort(byin.begin(), byin.end(), [&](int x, int y) { return d.in_pos[x] < d.in_pos[y]; });
    for (int r = 0; r < kTB; ++r) P.in_rank[byin[r]] = r;
    for (int b = 0; b < kTB; ++b) P.out_pos[b] = d.out_pos[b];
    // map 0: window = tile bits 0..4, thread bits by input position (coalesced landing reads)
    {
        std::vector<int> rest;
        for (int r = 0; r < kTB; ++r)
            if (byin[r] >= kWB) rest.push_back(byin[r]);
        for (int t = 0; t < kThrBits; ++t) P.order0[t] = rest[t];
    }
    // map 1: window = tile bits a-5..a-1, thread bits by output position
    // (coalesced stores; global tile bits, out_pos -1, last)
    {
        std::vector<int> rest;
        for (int b = 0; b < kTB; ++b)
            if (b < d.a - kWB || b >= d.a) rest.push_back(b);
        auto key = [&](int b) { return d.out_pos[b] < 0 ? 1000 + b : d.out_pos[b]; };
        std::sort(rest.begin(), rest.end(), [&](int x, int y) { return key(x) < key(y); });
        for (int t = 0; t < kThrBits; ++t) P.order1[t] = rest[t];
    }
    // rank-group pass: the global tile bits (in_pos >= nl) are the highest-ranked
    P.ng = d.ng;
    for (int i = 0; i < d.ng; ++i) {
        if (byin[kTB - d.ng + i] != d.gbit[i] || d.in_pos[d.gbit[i]] < nl) return false;
        P.split_bit[i] = d.split_fix[i];
        P.gthr[i] = P.gwin[i] = -1;
        for (int t = 0; t < kThrBits; ++t)
            if (P.order1[t] == d.gbit[i]) P.gthr[i] = t;
        if (d.gbit[i] >= d.a - kWB && d.gbit[i] < d.a) P.gwin[i] = d.gbit[i] - (d.a - kWB);
    }
    P.split_val = d.split_val;
    for (int c = 0; c < (1 << d.ng); ++c) P.outb[c] = d.gbase[c];
    // early wires: on tile bits they must be thread bits of map 0 (they are passive bits >= a)
    P.n_et = d.n_et;
    for (int e = 0; e < d.n_et; ++e) {
        if (d.et_bit[e] < kWB) return false;
        P.et_bit[e] = d.et_bit[e];
        P.et_w[e] = d.et_w[e];
    }
    P.n_ef = d.n_ef;
    // runs of consecutive (tile-id bit, target bit) pairs
    auto runs = [](int cnt, const int *src, const int *dst, int &n, int *rs, int *rl, int *rd) {
        std::vector<std::pair<int, int>> v;
        for (int i = 0; i < cnt; ++i) v.push_back({src[i], dst[i]});
        std::sort(v.begin(), v.end());
        n = 0;
        for (size_t i = 0; i < v.size(); ++i) {
            if (n > 0 && v[i].first == rs[n - 1] + rl[n - 1] && v[i].second == rd[n - 1] + rl[n - 1]) {
                rl[n - 1]++;
                continue;
            }
            rs[n] = v[i].first;
            rl[n] = 1;
            rd[n] = v[i].second;
            n++;
        }
    };
    runs(d.n_ef, d.ef_bit, d.ef_w, P.n_erun, P.erun_src, P.erun_len, P.erun_dst);
    {
        std::vector<int> fidx(d.nfix);
        for (int f = 0; f < d.nfix; ++f) fidx[f] = f;
        runs(d.nfix, fidx.data(), d.fout_pos, P.n_orun, P.orun_src, P.orun_len, P.orun_dst);
    }
    P.y_const = d.y_const;
    // a window-1 bit on output position 0: each thread holds neighbouring
    // pairs, stored 32 bytes at a time (QSIM_NO_ST256: 16-byte stores)
    static const bool no_st256 = getenv("QSIM_NO_ST256") != nullptr;   // measurement knob
    P.pb = -1;
    for (int b = 0; b < kWB && !no_st256 && d.ng == 0; ++b)
        if (d.out_pos[d.a - kWB + b] == 0) P.pb = b;
    P.nfix = d.nfix;
    // quarter boxes: the 11 lowest-ranked tile bits form the box; the two
    // highest-ranked tile bits join the fixed positions as "ext-id" bits
    std::vector<int> sub_pos;
    for (int r = 0; r < kQB; ++r) sub_pos.push_back(d.in_pos[byin[r]]);
    std::vector<int> fid(nl, -1);
    {
        std::vector<char> in_sub(nl, 0);
        for (int p : sub_pos) {
            if (p >= nl) return false;
            in_sub[p] = 1;
        }
        int e = 0;
        P.qe0 = P.qe1 = -1;
        for (int p = 0; p < nl; ++p) {
            if (in_sub[p]) continue;
            if (p == d.in_pos[byin[kQB]]) P.qe0 = e;
            if (p == d.in_pos[byin[kQB + 1]]) P.qe1 = e;
            fid[p] = e++;
        }
        // local quarter bits are ext-id bits; global ones (rank-group pass) pick the shard
        if ((d.ng < 2 && P.qe0 < 0) || (d.ng < 1 && P.qe1 < 0) || (P.qe1 >= 0 && P.qe0 > P.qe1)) return false;
        // the tile-id bits fill the other ext bits in ascending position order,
        // which is the order of d.fin_pos (ascending)
        for (int f = 1; f < d.nfix; ++f)
            if (d.fin_pos[f] < d.fin_pos[f - 1]) return false;
    }
    CUtensorMap im[4];
    int rank_sub[kQB];
    std::memset(im, 0, sizeof im);
    for (int c = 0; c < (1 << d.ng); ++c)
        if (!build_side(d.ng ? d.gbase[c] : in, nl, sub_pos, fid, im[c], P.in_first, P.in_len, rank_sub))
            return false;
    const uint64_t ntiles = 1ull << (d.nfix - d.ng);   // this rank's share of the tiles
    switch (d.a) {
    case 5: launch13_a<5>(h, im, out, P, ntiles, d.inverse, d.hadamard_only); break;
    case 6: launch13_a<6>(h, im, out, P, ntiles, d.inverse, d.hadamard_only); break;
    case 7: launch13_a<7>(h, im, out, P, ntiles, d.inverse, d.hadamard_only); break;
    case 8: launch13_a<8>(h, im, out, P, ntiles, d.inverse, d.hadamard_only); break;
    case 9: launch13_a<9>(h, im, out, P, ntiles, d.inverse, d.hadamard_only); break;
    default: launch13_a<10>(h, im, out, P, ntiles, d.inverse, d.hadamard_only); break;
    }
    return true;
}

}  // namespace qs
