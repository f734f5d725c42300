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
__device__ __forceinline__ double2 root_of_unity(uint64_t t, int W, const double2 *tab, int inverse)
{
    if (W <= 10) return tab[(uint32_t)(t << (10 - W)) & 1023u];
    const uint64_t hi = t >> (W - 10);
    const uint64_t lo = t & ((1ull << (W - 10)) - 1);
    double2 p = tab[(uint32_t)hi & 1023u];
    if (lo) {
        // theta = 2 pi lo / 2^W
        double th = (double)lo * ldexp(6.283185307179586476925286766559, -W);
        if (inverse) th = -th;
        const double t2 = th * th;
        const double c = fma(fma(fma(-t2, 1.0 / 720.0, 1.0 / 24.0), t2, -0.5), t2, 1.0);
        const double s = th * fma(fma(fma(-t2, 1.0 / 5040.0, 1.0 / 120.0), t2, -1.0 / 6.0), t2, 1.0);
        p = cmul(p, make_double2(c, s));
    }
    return p;
}

__global__ void __launch_bounds__(512) k_tile_pass(const __grid_constant__ TilePass tp,
                                                   const double2 *in, double2 *out, uint64_t ntiles)
{
    extern __shared__ double2 smem[];
    double2 *tile = smem;
    double2 *tab = smem + (1u << tp.tbits);
    const uint32_t tid = threadIdx.x;
    const int tb = tp.tbits - kRegBits;   // thread bits

    // roots of unity exp(+-2 pi i k / 1024)
    for (uint32_t k = tid; k < 1024; k += blockDim.x) {
        double s, c;
        sincospi((double)k / 512.0, &s, &c);
        tab[k] = make_double2(c, tp.inverse ? -s : s);
    }
    __syncthreads();

    const TileMap &m0 = tp.map[0];
    const TileMap &mL = tp.map[tp.nmaps - 1];
    // per-thread parts of the load / store offsets (tile-local -> position offsets)
    uint64_t tin = 0, tout = 0;
    for (int t = 0; t < tb; ++t) {
        const uint64_t bit = (tid >> t) & 1u;
        tin |= bit << tp.in_pos[m0.order[t]];
        tout |= bit << tp.out_pos[mL.order[t]];
    }
    uint64_t pin[kRegBits], pout[kRegBits];
#pragma unroll
    for (int b = 0; b < kRegBits; ++b) {
        pin[b] = 1ull << tp.in_pos[m0.win[b]];
        pout[b] = 1ull << tp.out_pos[mL.win[b]];
    }

    const uint32_t amask = (1u << tp.a) - 1u;

    for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        uint64_t ib = 0, ob = 0;
        for (int f = 0; f < tp.nfix; ++f) {
            const uint64_t bit = (T >> f) & 1u;
            ib |= bit << tp.fin_pos[f];
            ob |= bit << tp.fout_pos[f];
        }
        uint64_t yfix = tp.y_const;
        for (int e = 0; e < tp.n_ef; ++e) yfix += ((T >> tp.ef_bit[e]) & 1u) << tp.ef_w[e];

        double2 v[NS];
        // ---- gather (map 0)
        {
            const uint64_t base = ib | tin;
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                uint64_t o = 0;
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
                    if (k & (1 << b)) o |= pin[b];
                v[k] = __ldcs(in + (base | o));
            }
        }
        // ---- twiddle + normalisation (before any H of this pass)
        {
            uint32_t wb[kRegBits];
#pragma unroll
            for (int b = 0; b < kRegBits; ++b) wb[b] = 1u << m0.win[b];
            const uint32_t tpart = thread_part(m0, tb, tid);
            const bool has_y = !tp.hadamard_only && (tp.n_et > 0 || tp.n_ef > 0 || tp.y_const != 0);
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                uint32_t ti = tpart;
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
                    if (k & (1 << b)) ti |= wb[b];
                double2 ph = make_double2(tp.scale, 0.0);
                if (has_y && tp.a > 0) {
                    uint64_t Y = yfix;
                    for (int e = 0; e < tp.n_et; ++e) Y += (uint64_t)((ti >> tp.et_bit[e]) & 1u) << tp.et_w[e];
                    const uint32_t J = __brev(ti & amask) >> (32 - tp.a);
                    const uint64_t t = Y * (uint64_t)J;
                    if (t) {
                        const double2 r = root_of_unity(t, tp.W, tab, tp.inverse);
                        ph = make_double2(r.x * tp.scale, r.y * tp.scale);
                    }
                }
                v[k] = cmul(v[k], ph);
            }
        }
        // ---- register windows
        for (int mi = 0; mi < tp.nmaps; ++mi) {
            const TileMap &m = tp.map[mi];
            uint32_t wb[kRegBits];
#pragma unroll
            for (int b = 0; b < kRegBits; ++b) wb[b] = 1u << m.win[b];
            const uint32_t tpart = thread_part(m, tb, tid);
            if (mi > 0) {
                const TileMap &pm = tp.map[mi - 1];
                uint32_t pwb[kRegBits];
#pragma unroll
                for (int b = 0; b < kRegBits; ++b) pwb[b] = 1u << pm.win[b];
                const uint32_t ptpart = thread_part(pm, tb, tid);
                __syncthreads();   // previous readers of the tile buffer are done
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    uint32_t ti = ptpart;
#pragma unroll
                    for (int b = 0; b < kRegBits; ++b)
                        if (k & (1 << b)) ti |= pwb[b];
                    tile[swz(ti)] = v[k];
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    uint32_t ti = tpart;
#pragma unroll
                    for (int b = 0; b < kRegBits; ++b)
                        if (k & (1 << b)) ti |= wb[b];
                    v[k] = tile[swz(ti)];
                }
            }
            if (m.ucnt > 0) {
                const int w0 = m.win[0];   // compute windows are contiguous: win[b] = w0 + b
#pragma unroll
                for (int rb = 0; rb < kRegBits; ++rb) {
                    const int u = w0 + rb;
                    if (u < m.ustart || u >= m.ustart + m.ucnt) continue;
                    // phase exp(i pi sum_{u'<u} y_u' 2^(u'-u)) on b_u = 1
                    if (u > 0 && !tp.hadamard_only) {
                        const uint32_t zmask = (1u << u) - 1u;
#pragma unroll
                        for (int k = 0; k < NS; ++k) {
                            if (!(k & (1 << rb))) continue;
                            uint32_t ti = tpart;
#pragma unroll
                            for (int b = 0; b < kRegBits; ++b)
                                if (k & (1 << b)) ti |= wb[b];
                            const uint32_t z = ti & zmask;
                            if (z) v[k] = cmul(v[k], tab[(z << (9 - u)) & 1023u]);
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
        // ---- scatter (last map)
        {
            const uint64_t base = ob | tout;
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                uint64_t o = 0;
#pragma unroll
                for (int b = 0; b < kRegBits; ++b)
                    if (k & (1 << b)) o |= pout[b];
                __stcs(out + (base | o), v[k]);
            }
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

void launch_tile_pass(Handle *h, const TilePass &tp, const double2 *in, double2 *out)
{
    const size_t smem = (sizeof(double2) << tp.tbits) + 1024 * sizeof(double2);
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(k_tile_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((sizeof(double2) << kTileMaxBits) + 1024 * sizeof(double2)));
        attr_done = true;
    }
    const int threads = 1 << (tp.tbits - kRegBits);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile_pass, threads, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t ntiles = 1ull << tp.nfix;
    const uint64_t cap = (uint64_t)h->num_sms * per_sm;
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    prof_begin(h);
    k_tile_pass<<<grid, threads, smem, h->stream>>>(tp, in, out, ntiles);
    prof_end(h, "k_tile_pass", (1ull << (tp.tbits + tp.nfix)) * 32);
}

}  // namespace qs
