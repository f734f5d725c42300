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
#include "tile_common.cuh"

#include <algorithm>

namespace qs {

namespace {

using namespace tile;

// The pass kernel.  NM = number of register maps (compile time, so that all
// per-map values live in registers and every slot index is static).
template <int NM>
__global__ void __launch_bounds__(1 << (kTileMaxBits - kRegBits), 1) k_tile_pass(const __grid_constant__ TilePass tp,
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
        tile_body<NM, false>(v, tp, tpart, stp, tab, tile, T, yt, Jt, twid, amask, sg);
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
        // the last window ends at the last active wire (already transformed
        // wires fill it up) so that passive tile bits stay thread bits: the
        // gather / scatter maps then walk the lowest positions
        int w0 = s * kRegBits;
        if (w0 + kRegBits > tp.a) w0 = std::max(0, tp.a - kRegBits);
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
    static uint64_t attr_done = 0;
    if (first_use_on_device(attr_done)) {
        cudaFuncSetAttribute(k_tile_pass<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((sizeof(double2) << kTileMaxBits) + 1024 * sizeof(double2)));
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

void finish_tile_pass(TilePass &tp)
{
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
}

void launch_tile_pass(Handle *h, const TilePass &tp_in, const double2 *in, double2 *out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    if (launch_tile_pass_tma(h, tp_in, in, out)) return;
    TilePass tp = tp_in;
    finish_tile_pass(tp);
    switch (tp.nmaps) {
    case 1: launch_nm<1>(h, tp, in, out); break;
    case 2: launch_nm<2>(h, tp, in, out); break;
    case 3: launch_nm<3>(h, tp, in, out); break;
    case 4: launch_nm<4>(h, tp, in, out); break;
    case 5: launch_nm<5>(h, tp, in, out); break;
    default: launch_nm<6>(h, tp, in, out); break;
    }
}

}  // namespace qs
