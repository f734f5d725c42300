// k_gates.cu -- unfused streaming gate kernels on one shard (sm_100a).
//
// Each kernel is the paper's in-place pair update (§2.2.1)
// mapped to the GPU: one thread owns a set of amplitude pairs (j, j + 2^p)
// for the whole update, so the "temporary t1" of the paper lives in a
// register and no barrier is needed; the barrier between gates is stream
// order.  Pair indices are produced by inserting a zero bit at position p
// into a dense counter, so every thread has work (no idle half of the index
// space) and a warp reads 32 consecutive 16-byte amplitudes for both members
// of the pair when p >= 5 (two fully used 512-byte segments).  These kernels
// are HBM-bound: 32 bytes per amplitude pair per gate (read + write).
#include "qsim_internal.h"

namespace qs {

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;   // pairs per thread per iteration (memory-level parallelism)

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma2(double2 u, double2 x, double2 v, double2 y)
{
    // u*x + v*y
    double re = fma(u.x, x.x, -u.y * x.y);
    double im = fma(u.x, x.y, u.y * x.x);
    re = fma(v.x, y.x, re);
    re = fma(-v.y, y.y, re);
    im = fma(v.x, y.y, im);
    im = fma(v.y, y.x, im);
    return make_double2(re, im);
}

__device__ __forceinline__ uint64_t insert_zero(uint64_t j, int p)
{
    const uint64_t lo = j & ((1ull << p) - 1);
    return ((j >> p) << (p + 1)) | lo;
}

struct Mat { double2 u[4]; };

// Dense 2x2 (u11 u12; u21 u22) on position p, where (i0 & cm) == cv.
__global__ void __launch_bounds__(kThreads) k_apply_2x2(double2 *__restrict__ psi, uint64_t npairs,
                                                        int p, uint64_t cm, uint64_t cv, Mat U)
{
    const uint64_t s = 1ull << p;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < npairs;
         base += stride * kUnroll) {
        double2 a[kUnroll], b[kUnroll];
        uint64_t i0[kUnroll];
        bool ok[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const uint64_t j = base + (uint64_t)k * stride;
            i0[k] = insert_zero(j, p);
            ok[k] = j < npairs && (i0[k] & cm) == cv;
            if (ok[k]) { a[k] = __ldcs(psi + i0[k]); b[k] = __ldcs(psi + i0[k] + s); }
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            if (!ok[k]) continue;
            const double2 x = cfma2(U.u[0], a[k], U.u[1], b[k]);
            const double2 y = cfma2(U.u[2], a[k], U.u[3], b[k]);
            __stcs(psi + i0[k], x);
            __stcs(psi + i0[k] + s, y);
        }
    }
}

// Multiply amplitudes with (i & mask) == val by ph; enumerates only those.
// mask bits are inserted in ascending order (nb <= 64 bits of mask).
struct MaskBits { int nb; int bit[40]; };
__global__ void __launch_bounds__(kThreads) k_phase_mask(double2 *__restrict__ psi, uint64_t count,
                                                         MaskBits mb, uint64_t val, double2 ph)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
        uint64_t i = j;
        for (int k = 0; k < mb.nb; ++k) i = insert_zero(i, mb.bit[k]);
        i |= val;
        __stcs(psi + i, cmul(__ldcs(psi + i), ph));
    }
}

// Swap local positions p1 < p2: exchange |..1..0..> and |..0..1..>.
__global__ void __launch_bounds__(kThreads) k_swap(double2 *__restrict__ psi, uint64_t count, int p1,
                                                   int p2)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
        uint64_t i = insert_zero(insert_zero(j, p1), p2);
        const uint64_t a = i | (1ull << p1), b = i | (1ull << p2);
        const double2 t = psi[a];
        psi[a] = psi[b];
        psi[b] = t;
    }
}

__global__ void __launch_bounds__(kThreads) k_scale(double2 *__restrict__ psi, uint64_t count, double s)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
        double2 v = psi[j];
        psi[j] = make_double2(v.x * s, v.y * s);
    }
}

// A 2x2 gate on a qubit that sits on a rank bit, computed in one kernel over
// peer memory (SURVEY §8(e) fused alternative): the partner rank holds the
// other row of every pair at the same local index, so this rank's output is
// out_i = a * mine_i + c * theirs_i (a, c = this rank's row of U), reading
// `theirs` straight from the partner's shard over NVLink -- the exchange and
// the gate are one pass (16 B read local + 16 B read remote + 16 B written per
// amplitude).  Amplitudes failing the local controls are copied.
__global__ void __launch_bounds__(kThreads) k_apply_2x2_remote(const double2 *__restrict__ mine,
                                                               const double2 *__restrict__ theirs,
                                                               double2 *__restrict__ out, uint64_t count,
                                                               uint64_t cm, uint64_t cv, double2 a, double2 c)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const double2 x = __ldcs(mine + i);
        if ((i & cm) == cv) {
            const double2 y = __ldcs(theirs + i);
            __stcs(out + i, cfma2(a, x, c, y));
        } else {
            __stcs(out + i, x);
        }
    }
}

__global__ void k_set_one(double2 *psi, uint64_t i) { psi[i] = make_double2(1.0, 0.0); }

}  // namespace

static unsigned grid_for(const Handle *h, uint64_t work)
{
    const uint64_t want = (work + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)h->num_sms * 8;   // resident: 8 x 256 threads per SM
    return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

void launch_apply_2x2(Handle *h, int p, uint64_t cm, uint64_t cv, const double2 U[4])
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    Mat m;
    for (int k = 0; k < 4; ++k) m.u[k] = U[k];
    const uint64_t np = h->local_dim() >> 1;
    prof_begin(h);
    k_apply_2x2<<<grid_for(h, (np + kUnroll - 1) / kUnroll), kThreads, 0, h->stream>>>(h->psi, np, p,
                                                                                      cm, cv, m);
    prof_end(h, "k_apply_2x2", (np >> __builtin_popcountll(cm)) * 64);   // 2 amplitudes read + written per pair
}

void launch_apply_diag(Handle *h, int p, uint64_t cm, uint64_t cv, double2 d0, double2 d1)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    // diag(d0, d1) = two masked phase multiplications (skip the identity halves)
    const bool one0 = d0.x == 1.0 && d0.y == 0.0, one1 = d1.x == 1.0 && d1.y == 0.0;
    const uint64_t bit = 1ull << p;
    if (!one0) launch_phase_mask(h, cm | bit, cv, d0);
    if (!one1) launch_phase_mask(h, cm | bit, cv | bit, d1);
}

void launch_phase_mask(Handle *h, uint64_t mask, uint64_t val, double2 ph)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    MaskBits mb;
    mb.nb = 0;
    for (int b = 0; b < h->nl; ++b)
        if ((mask >> b) & 1) mb.bit[mb.nb++] = b;
    const uint64_t count = h->local_dim() >> mb.nb;
    prof_begin(h);
    k_phase_mask<<<grid_for(h, count), kThreads, 0, h->stream>>>(h->psi, count, mb, val & mask, ph);
    prof_end(h, "k_phase_mask", count * 32);
}

void launch_swap_local(Handle *h, int p1, int p2)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    if (p1 == p2) return;
    if (p1 > p2) { int t = p1; p1 = p2; p2 = t; }
    const uint64_t count = h->local_dim() >> 2;
    prof_begin(h);
    k_swap<<<grid_for(h, count), kThreads, 0, h->stream>>>(h->psi, count, p1, p2);
    prof_end(h, "k_swap", count * 64);
}

void launch_scale(Handle *h, double s)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const uint64_t count = h->local_dim();
    prof_begin(h);
    k_scale<<<grid_for(h, count), kThreads, 0, h->stream>>>(h->psi, count, s);
    prof_end(h, "k_scale", count * 32);
}

void launch_zero(Handle *h)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    cudaMemsetAsync(h->psi, 0, sizeof(double2) * h->local_dim(), h->stream);
}

void launch_apply_2x2_remote(Handle *h, const double2 *theirs, double2 *out, uint64_t cm, uint64_t cv, double2 a,
                             double2 c)
{
    cudaSetDevice(h->device);
    const uint64_t count = h->local_dim();
    const uint64_t matching = count >> __builtin_popcountll(cm);
    prof_begin(h);
    k_apply_2x2_remote<<<grid_for(h, count), kThreads, 0, h->stream>>>(h->psi, theirs, out, count, cm, cv, a, c);
    prof_end(h, "k_apply_2x2_remote", count * 32 + matching * 16);
}

void launch_set_one(Handle *h, uint64_t local_idx)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    prof_begin(h);
    k_set_one<<<1, 1, 0, h->stream>>>(h->psi, local_idx);
    prof_end(h, "k_set_one", 16);
}

}  // namespace qs
