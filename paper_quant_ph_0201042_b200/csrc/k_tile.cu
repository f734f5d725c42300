// k_tile.cu -- fused QFT passes and bit-permutation passes (sm_100a).
//
// The QFT circuit (§2.3.2: H(j), then R_{k-j} controlled by
// k on target j for k > j, then the closing swaps) is applied in a few HBM
// passes instead of one pass per gate.  The wires are cut into consecutive
// blocks A = {a0 .. a0+a-1}; one pass applies every gate that touches A:
//
//   * R_d gates are diagonal, so each R_{j-i}(i < j) may be applied anywhere
//     between H(i) and H(j).  We apply it right before H(j).  For i in an
//     earlier block those phases depend only on the (already transformed)
//     early wires and on the computational bit of j, and no gate of this
//     pass touches the early wires, so all of them are applied at the start
//     of the pass as one "twiddle" exp(2 pi i Y J / 2^W), Y = sum_{i<a0}
//     y_i 2^i, J = sum_{j in A} b_j 2^(a0+a-1-j), W = a0+a  (this is exactly
//     the Cooley-Tukey twiddle of the QFT's FFT structure);
//   * inside A, before H(j) the amplitudes with b_j = 1 get
//     exp(i pi sum_{i in A, i<j} y_i 2^(i-j)) from a 1024-entry table of
//     roots of unity, then H(j) acts on the register pair (unnormalised;
//     the 2^(-a/2) is folded into the twiddle);
//   * the closing swaps are a relabelling of wires, folded into the store
//     addresses of the pass (out_pos).
//
// A tile holds 2^tbits amplitudes (the active wires + "passive" low
// positions so that every gather/scatter moves runs of >= 2^L contiguous
// amplitudes).  Each thread keeps 16 amplitudes in registers; four wires are
// processed per register window; windows change through shared memory
// (XOR-swizzled, 16-byte accesses).  Work per amplitude per pass: one HBM
// read + write (32 B), ~4 FP64 ops per active wire plus one twiddle.
#include "qsim_internal.h"

#include <algorithm>

namespace qs {

namespace {

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

// The pass kernel.  NM = number of register maps (compile time, so that all
// per-map values live in registers and every slot index is static).
template <int NM>
__global__ void __launch_bounds__(256, 1) k_tile_pass(const __grid_constant__ TilePass tp,
                                                   const double2 *in, double2 *out, uint64_t ntiles)
{
    extern __shared__ double2 smem[];
    double2 *tile = smem;
    double2 *tab = smem + (1u << tp.tbits);
    const uint32_t tid = threadIdx.x;
    const int tb = tp.tbits - kRegBits;   // thread bits
    const double sg = tp.inverse ? -1.0 : 1.0;

    // roots of unity exp(+-2 pi i k / 1024)
    for (uint32_t k = tid; k < 1024; k += blockDim.x) {
        double s, c;
        sincospi((double)k / 512.0, &s, &c);
        tab[k] = make_double2(c, sg * s);
    }
    __syncthreads();

    // per-thread constants (all maps)
    uint32_t tpart[NM], stp[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        tpart[m] = thread_part(tp.map[m], tb, tid);
        stp[m] = swz(tpart[m]);
    }
    uint64_t tin = 0, tout = 0;
    for (int t = 0; t < tb; ++t) {
        const uint64_t bit = (tid >> t) & 1u;
        tin |= bit << tp.in_pos[tp.map[0].order[t]];
        tout |= bit << tp.out_pos[tp.map[NM - 1].order[t]];
    }
    uint64_t pin[kRegBits], pout[kRegBits];
#pragma unroll
    for (int b = 0; b < kRegBits; ++b) {
        pin[b] = 1ull << tp.in_pos[tp.map[0].win[b]];
        pout[b] = 1ull << tp.out_pos[tp.map[NM - 1].win[b]];
    }
    const bool twid = !tp.hadamard_only && tp.a > 0 && (tp.n_et > 0 || tp.n_ef > 0 || tp.y_const != 0);
    const uint32_t amask = (1u << tp.a) - 1u;
    const uint32_t Jt = tp.a > 0 ? (__brev(tpart[0] & amask) >> (32 - tp.a)) : 0u;
    uint64_t yt = 0;
    for (int e = 0; e < tp.n_et; ++e) yt += (uint64_t)((tpart[0] >> tp.et_bit[e]) & 1u) << tp.et_w[e];

    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        uint64_t ib = 0, ob = 0;
        for (int f = 0; f < tp.nfix; ++f) {
            const uint64_t bit = (T >> f) & 1u;
            ib |= bit << tp.fin_pos[f];
            ob |= bit << tp.fout_pos[f];
        }
        double2 v[NS];
        // ---- gather (map 0): lowest thread bits walk the lowest input positions
        {
            uint64_t o[NS];
            o[0] = ib | tin;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int j = 0; j < (1 << b); ++j) o[j | (1 << b)] = o[j] | pin[b];
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k] = __ldcs(in + o[k]);
        }
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
                __syncthreads();   // previous readers of the tile buffer are done
#pragma unroll
                for (int k = 0; k < NS; ++k) tile[s[k]] = v[k];
                s[0] = stp[m];
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                    for (int j = 0; j < (1 << b); ++j) s[j | (1 << b)] = s[j] ^ tp.wswz[m][b];
                __syncthreads();
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
        // ---- scatter (last map): lowest thread bits walk the lowest output positions
        {
            uint64_t o[NS];
            o[0] = ob | tout;
#pragma unroll
            for (int b = 0; b < kRegBits; ++b)
#pragma unroll
                for (int j = 0; j < (1 << b); ++j) o[j | (1 << b)] = o[j] | pout[b];
#pragma unroll
            for (int k = 0; k < NS; ++k) __stcs(out + o[k], v[k]);
        }
    }
}

}  // namespace

// ------------------------------------------------------------------ host planning

// Fill tp.map[] (register windows, thread orders) from tbits / a / in_pos /
// out_pos.  Map 0 gathers (its lowest thread bits walk the lowest input
// positions), the last map scatters (lowest thread bits walk the lowest
// output positions); compute maps hold four consecutive active wires.
void plan_tile_maps(TilePass &tp)
{
    const int tb = tp.tbits - kRegBits;
    auto order_by = [&](TileMap &m, const int *key) {
        std::vector<int> rest;
        for (int b = 0; b < tp.tbits; ++b) {
            bool inw = false;
            for (int k = 0; k < kRegBits; ++k) inw |= m.win[k] == b;
            if (!inw) rest.push_back(b);
        }
        if (key) std::stable_sort(rest.begin(), rest.end(), [&](int x, int y) { return key[x] < key[y]; });
        for (int t = 0; t < tb; ++t) m.order[t] = rest[t];
    };
    auto io_map = [&](TileMap &m, const int *key) {   // window = the 4 highest positions
        std::vector<int> bits(tp.tbits);
        for (int b = 0; b < tp.tbits; ++b) bits[b] = b;
        std::stable_sort(bits.begin(), bits.end(), [&](int x, int y) { return key[x] > key[y]; });
        for (int k = 0; k < kRegBits; ++k) m.win[k] = bits[kRegBits - 1 - k];
        order_by(m, key);
        m.ustart = 0;
        m.ucnt = 0;
    };
    // a map moves runs well for `key` if its first thread bits are the 3
    // lowest positions of the whole tile, in order
    auto good_for = [&](const TileMap &m, const int *key) {
        std::vector<int> all(tp.tbits);
        for (int b = 0; b < tp.tbits; ++b) all[b] = key[b];
        std::sort(all.begin(), all.end());
        const int L = std::min(3, tb);
        for (int t = 0; t < L; ++t)
            if (key[m.order[t]] != all[t]) return false;
        return true;
    };
    std::vector<TileMap> maps;
    const int nstage = (tp.a + kRegBits - 1) / kRegBits;
    for (int s = 0; s < nstage; ++s) {
        TileMap m;
        int w0 = s * kRegBits;
        if (w0 + kRegBits > tp.tbits) w0 = tp.tbits - kRegBits;
        for (int k = 0; k < kRegBits; ++k) m.win[k] = w0 + k;
        m.ustart = s * kRegBits;
        m.ucnt = std::min(tp.a, (s + 1) * kRegBits) - s * kRegBits;
        order_by(m, s == 0 ? tp.in_pos : (s == nstage - 1 ? tp.out_pos : nullptr));
        maps.push_back(m);
    }
    if (maps.empty() || !good_for(maps.front(), tp.in_pos)) {
        TileMap l;
        io_map(l, tp.in_pos);
        maps.insert(maps.begin(), l);
    }
    bool moved = false;
    for (int b = 0; b < tp.tbits; ++b) moved |= tp.in_pos[b] != tp.out_pos[b];
    if (maps.size() == 1 ? (moved || !good_for(maps.back(), tp.out_pos))
                         : !good_for(maps.back(), tp.out_pos)) {
        TileMap l;
        io_map(l, tp.out_pos);
        maps.push_back(l);
    }
    tp.nmaps = (int)maps.size();
    for (int i = 0; i < tp.nmaps; ++i) tp.map[i] = maps[i];
}

static uint32_t swz_host(uint32_t ti)
{
    uint32_t f = (ti >> 3) ^ (ti >> 6) ^ (ti >> 9) ^ (ti >> 12);
    return ti ^ (f & 7u);
}

template <int NM>
static void launch_nm(Handle *h, const TilePass &tp, const double2 *in, double2 *out)
{
    const size_t smem = (sizeof(double2) << tp.tbits) + 1024 * sizeof(double2);
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(k_tile_pass<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((sizeof(double2) << kTileMaxBits) + 1024 * sizeof(double2)));
        attr_done = true;
    }
    const int threads = 1 << (tp.tbits - kRegBits);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile_pass<NM>, threads, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t ntiles = 1ull << tp.nfix;
    const uint64_t cap = (uint64_t)h->num_sms * per_sm;
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    prof_begin(h);
    k_tile_pass<NM><<<grid, threads, smem, h->stream>>>(tp, in, out, ntiles);
    prof_end(h, "k_tile_pass", (1ull << (tp.tbits + tp.nfix)) * 32);
}

void launch_tile_pass(Handle *h, const TilePass &tp_in, const double2 *in, double2 *out)
{
    TilePass tp = tp_in;
    // derived constants (host side): swizzled window bits, J weights of the
    // map-0 window, whether every early tile bit is a thread bit of map 0
    for (int m = 0; m < tp.nmaps; ++m)
        for (int b = 0; b < kRegBits; ++b) tp.wswz[m][b] = swz_host(1u << tp.map[m].win[b]);
    for (int b = 0; b < kRegBits; ++b) {
        const int w = tp.map[0].win[b];
        tp.jwin[b] = w < tp.a ? (1u << (tp.a - 1 - w)) : 0u;
    }
    tp.twiddle_fast = 1;
    for (int e = 0; e < tp.n_et; ++e)
        for (int b = 0; b < kRegBits; ++b) tp.twiddle_fast &= tp.et_bit[e] != tp.map[0].win[b];
    tp.tw = (tp.inverse ? -1.0 : 1.0) * 6.283185307179586476925286766559 / std::ldexp(1.0, tp.W);
    switch (tp.nmaps) {
    case 1: launch_nm<1>(h, tp, in, out); break;
    case 2: launch_nm<2>(h, tp, in, out); break;
    case 3: launch_nm<3>(h, tp, in, out); break;
    case 4: launch_nm<4>(h, tp, in, out); break;
    default: launch_nm<5>(h, tp, in, out); break;
    }
}

}  // namespace qs
