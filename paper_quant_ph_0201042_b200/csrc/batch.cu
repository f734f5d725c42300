// batch.cu -- batched noisy trajectories (DESIGN.md
// R33): the register of a trajectory is qubits [b, n) of the handle, the top
// b qubits (the MSBs, hence the rank bits of a sharded handle) index 2^b
// independent trajectories.  Trajectory t draws its gate noise from seed + t
// and its Pauli events from seed + t, so it is exactly the single-register
// circuit with that seed; gates with per-trajectory matrices read them from
// a device table indexed by t (GOP_DENSET in the fused passes).
//
// Kernels here: the per-trajectory angle-form matrices (Philox4x32-10 +
// Box-Muller + the U_R / U_P1 / U_P2 products of PAPER.md:542-569 on the
// device), the broadcast of one register state to every trajectory, and the
// per-trajectory overlap with a reference register (fidelity, PAPER.md:
// 1127-1128).
#include <cmath>

#include "philox.cuh"
#include "qsim_internal.h"

namespace qs {

namespace {

__device__ __forceinline__ double2 cm(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 ca(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

__device__ void mmul(const double2 A[4], const double2 B[4], double2 C[4])
{
    double2 r[4];
    r[0] = ca(cm(A[0], B[0]), cm(A[1], B[2]));
    r[1] = ca(cm(A[0], B[1]), cm(A[1], B[3]));
    r[2] = ca(cm(A[2], B[0]), cm(A[3], B[2]));
    r[3] = ca(cm(A[2], B[1]), cm(A[3], B[3]));
    for (int k = 0; k < 4; ++k) C[k] = r[k];
}
// U_R(t) = (cos -sin; sin cos), U_P1(p) = diag(1, e^{ip}), U_P2(p) = diag(e^{ip}, 1)
__device__ void ur(double t, double2 U[4])
{
    const double c = cos(t), s = sin(t);
    U[0] = make_double2(c, 0); U[1] = make_double2(-s, 0); U[2] = make_double2(s, 0); U[3] = make_double2(c, 0);
}
__device__ void up1(double p, double2 U[4])
{
    U[0] = make_double2(1, 0); U[1] = make_double2(0, 0); U[2] = make_double2(0, 0); U[3] = make_double2(cos(p), sin(p));
}
__device__ void up2(double p, double2 U[4])
{
    U[0] = make_double2(cos(p), sin(p)); U[1] = make_double2(0, 0); U[2] = make_double2(0, 0); U[3] = make_double2(1, 0);
}

// Angle-form matrix of gate g for trajectories [0, B): nominal angles plus
// sigma * z(draw(seed + t, OPNOISE, g, slot)) (R12-R15 with R33).
__global__ void k_batch_mats(int kind, double a0, double a1, double a2, double a3, double sigma, uint64_t seed,
                             uint64_t g, uint64_t B, double2 *__restrict__ out)
{
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= B) return;
    double a[4] = {a0, a1, a2, a3};
    const int na = kind == QSIM_GATE_RP ? 2 : kind == QSIM_GATE_P1 ? 1 : 4;
    for (int s = 0; s < na; ++s) {
        const u64x2 d = draw(seed + t, QSIM_TAG_OPNOISE, g, (uint32_t)s);
        const double z = sqrt(-2.0 * log(u01o(d.a))) * cos(2.0 * M_PI * u01(d.b));
        a[s] += sigma * z;
    }
    double2 A[4], Bm[4], C[4], U[4];
    if (kind == QSIM_GATE_RP) {
        ur(a[0], A); up1(a[1], Bm); mmul(A, Bm, U);
    } else if (kind == QSIM_GATE_P1) {
        up1(a[0], U);
    } else {
        up2(a[0], A); up1(a[1], Bm); mmul(A, Bm, C);
        ur(a[2], A); mmul(C, A, Bm);
        up1(a[3], A); mmul(Bm, A, U);
    }
    for (int k = 0; k < 4; ++k) out[4 * t + k] = U[k];
}

// out[t] = B_t A_t: the product of two per-trajectory gates on one qubit
// (the planner merges runs of them into one table before a pass)
__global__ void k_batch_mul(double2 *__restrict__ out, const double2 *__restrict__ A, double2 a0, double2 a1,
                            double2 a2, double2 a3, const double2 *__restrict__ B, double2 b0, double2 b1, double2 b2,
                            double2 b3, uint64_t count)
{
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    double2 X[4] = {a0, a1, a2, a3}, Y[4] = {b0, b1, b2, b3}, Z[4];
    if (A)
        for (int k = 0; k < 4; ++k) X[k] = A[4 * t + k];
    if (B)
        for (int k = 0; k < 4; ++k) Y[k] = B[4 * t + k];
    mmul(Y, X, Z);
    for (int k = 0; k < 4; ++k) out[4 * t + k] = Z[k];
}

// psi[i] = src[i mod 2^r] * scale over the shard (every trajectory gets the
// same register state).
__global__ void __launch_bounds__(256) k_batch_broadcast(double2 *__restrict__ psi, uint64_t count,
                                                         const double2 *__restrict__ src, int r, double scale)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t mask = (1ull << r) - 1;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const double2 v = src[i & mask];
        psi[i] = make_double2(v.x * scale, v.y * scale);
    }
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// out[2 t], out[2 t + 1] = scale * sum_x conj(ref_x) psi[t 2^r + x] for the
// local trajectory t = blockIdx.x; fixed tree: per-thread contiguous runs,
// warp shuffles, then the block.
__global__ void __launch_bounds__(1024) k_batch_overlap(const double2 *__restrict__ psi,
                                                        const double2 *__restrict__ ref, int r, double scale,
                                                        double *__restrict__ out)
{
    __shared__ double sre[32], sim[32];
    const uint64_t len = 1ull << r;
    const double2 *p = psi + (uint64_t)blockIdx.x * len;
    const uint64_t per = (len + blockDim.x - 1) / blockDim.x;
    const uint64_t b = threadIdx.x * per;
    double re = 0.0, im = 0.0;
    for (uint64_t i = b; i < b + per && i < len; ++i) {
        const double2 x = ref[i], y = p[i];
        re = fma(x.x, y.x, fma(x.y, y.y, re));
        im = fma(x.x, y.y, fma(-x.y, y.x, im));
    }
    re = warp_sum(re);
    im = warp_sum(im);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sre[w] = re;
        sim[w] = im;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        re = l < nw ? sre[l] : 0.0;
        im = l < nw ? sim[l] : 0.0;
        re = warp_sum(re);
        im = warp_sum(im);
        if (l == 0) {
            out[2 * blockIdx.x] = re * scale;
            out[2 * blockIdx.x + 1] = im * scale;
        }
    }
}

}  // namespace

void launch_batch_mats(Handle *h, int kind, const double *ang, double sigma, uint64_t seed, uint64_t g, uint64_t B,
                       double2 *out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    double a[4] = {0, 0, 0, 0};
    const int na = kind == QSIM_GATE_RP ? 2 : kind == QSIM_GATE_P1 ? 1 : 4;
    for (int s = 0; s < na; ++s) a[s] = ang[s];
    prof_begin(h);
    k_batch_mats<<<(unsigned)((B + 127) / 128), 128, 0, h->stream>>>(kind, a[0], a[1], a[2], a[3], sigma, seed, g, B,
                                                                     out);
    prof_end(h, "k_batch_mats", B * 64);
}

void launch_batch_mul(Handle *h, double2 *out, const double2 *A, const double2 ac[4], const double2 *B,
                      const double2 bc[4], uint64_t count)
{
    cudaSetDevice(h->device);
    prof_begin(h);
    k_batch_mul<<<(unsigned)((count + 127) / 128), 128, 0, h->stream>>>(out, A, ac[0], ac[1], ac[2], ac[3], B, bc[0],
                                                                       bc[1], bc[2], bc[3], count);
    prof_end(h, "k_batch_mul", count * 192);
}

void launch_batch_broadcast(Handle *h, const double2 *src, int r, double scale)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const uint64_t count = h->local_dim();
    const uint64_t want = (count + 255) / 256;
    const uint64_t cap = (uint64_t)h->num_sms * 8;
    prof_begin(h);
    k_batch_broadcast<<<(unsigned)(want < cap ? want : cap), 256, 0, h->stream>>>(h->psi, count, src, r, scale);
    prof_end(h, "k_batch_broadcast", count * 16);
}

void launch_batch_overlap(Handle *h, const double2 *ref, int r, double scale, double *d_out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const uint64_t ntraj = h->local_dim() >> r;
    prof_begin(h);
    k_batch_overlap<<<(unsigned)ntraj, 1024, 0, h->stream>>>(h->psi, ref, r, scale, d_out);
    prof_end(h, "k_batch_overlap", h->local_dim() * 16 + ntraj * (16ull << r));
}

}  // namespace qs
