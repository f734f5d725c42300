// k_reduce.cu -- state preparation and read-out reductions (sm_100a).
//
// Reductions (norm, marginals, block sums for measurement) are read-only
// streaming passes: 16 bytes per amplitude.  Sums follow a fixed tree
// (per-thread sums of a few contiguous elements, warp shuffle tree, block
// tree, then a second-level tree over block partials), so results are
// deterministic and the rounding error grows like log(N), not sqrt(N)
// (R23).
#include "philox.cuh"
#include "qsim_internal.h"

namespace qs {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double abs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum (all threads must call); result valid in every thread.
__device__ double block_sum(double v, double *sh)
{
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    double t = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) sh[0] = t;
    __syncthreads();
    return sh[0];
}

// Sum of |a|^2 over chunks: block b sums [b*chunk, (b+1)*chunk) (chunk a
// multiple of blockDim) and writes out[b].
__global__ void __launch_bounds__(kThreads) k_chunk_abs2(const double2 *__restrict__ psi,
                                                         uint64_t chunk, double *__restrict__ out)
{
    __shared__ double sh[32];
    const uint64_t base = (uint64_t)blockIdx.x * chunk;
    double acc = 0.0;
    for (uint64_t i = threadIdx.x; i < chunk; i += blockDim.x) acc += abs2(psi[base + i]);
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// Tree sum of chunks of doubles: block b sums in[b*chunk .. b*chunk+count)
// (count <= chunk) and writes out[b]; each thread first sums a contiguous
// segment.
__global__ void __launch_bounds__(1024) k_sum_doubles(const double *__restrict__ in, uint64_t chunk,
                                                      uint64_t count, double *__restrict__ out)
{
    __shared__ double sh[32];
    in += (uint64_t)blockIdx.x * chunk;
    const uint64_t per = (count + blockDim.x - 1) / blockDim.x;
    double acc = 0.0;
    const uint64_t b = threadIdx.x * per;
    for (uint64_t i = b; i < b + per && i < count; ++i) acc += in[i];
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// Marginals when the sub-register occupies contiguous local positions
// [pl, pl+m): element i has value y = (i >> pl) & (2^m - 1).  Grid: one
// block per (y, rest-chunk); out[y * nchunk + c].
__global__ void __launch_bounds__(kThreads) k_probs_contig(const double2 *__restrict__ psi, int nl,
                                                           int pl, int m, uint64_t chunk,
                                                           uint64_t nchunk, double *__restrict__ out)
{
    __shared__ double sh[32];
    const uint64_t y = blockIdx.x / nchunk, c = blockIdx.x % nchunk;
    const uint64_t lowmask = (1ull << pl) - 1;
    double acc = 0.0;
    for (uint64_t r = c * chunk + threadIdx.x; r < (c + 1) * chunk; r += blockDim.x) {
        // r enumerates the bits outside [pl, pl+m): low pl bits, then the high ones
        const uint64_t i = ((r >> pl) << (pl + m)) | (y << pl) | (r & lowmask);
        acc += abs2(psi[i]);
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
    (void)nl;
}

// Marginals with one warp per value y (rest = 2^(nl-m) amplitudes per y, up
// to 2^14): grid-stride over y, lanes stride the y's amplitudes (16-byte
// loads, 512 contiguous bytes per warp load when the range sits above a
// contiguous low run), fixed xor tree; no per-y block and no finishing pass.
__global__ void __launch_bounds__(256) k_probs_warp(const double2 *__restrict__ psi, int pl, int m, uint64_t rest,
                                                    uint64_t ny, double *__restrict__ out)
{
    const uint64_t lowmask = (1ull << pl) - 1;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t y = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); y < ny; y += warps) {
        double acc0 = 0.0, acc1 = 0.0;
        uint64_t r = lane;
        for (; r + 32 < rest; r += 64) {
            const uint64_t i0 = ((r >> pl) << (pl + m)) | (y << pl) | (r & lowmask);
            const uint64_t r1 = r + 32;
            const uint64_t i1 = ((r1 >> pl) << (pl + m)) | (y << pl) | (r1 & lowmask);
            acc0 += abs2(psi[i0]);
            acc1 += abs2(psi[i1]);
        }
        if (r < rest) acc0 += abs2(psi[((r >> pl) << (pl + m)) | (y << pl) | (r & lowmask)]);
        const double s = warp_sum(acc0 + acc1);
        if (lane == 0) out[y] = s;
    }
}

// per-y tree over its chunks
__global__ void k_probs_finish(const double *__restrict__ part, uint64_t ny, uint64_t nchunk,
                               double *__restrict__ out)
{
    const uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= ny) return;
    // pairwise over nchunk (a power of two)
    double buf[64];
    uint64_t w = nchunk;
    if (w <= 64) {
        for (uint64_t c = 0; c < w; ++c) buf[c] = part[y * nchunk + c];
        while (w > 1) {
            for (uint64_t c = 0; c < w / 2; ++c) buf[c] = buf[2 * c] + buf[2 * c + 1];
            w /= 2;
        }
        out[y] = buf[0];
    } else {
        double s = 0.0;
        for (uint64_t c = 0; c < nchunk; ++c) s += part[y * nchunk + c];
        out[y] = s;
    }
}

// <a|b> over chunks: block c sums conj(a_i) b_i over [c*chunk, (c+1)*chunk)
// and writes re to out_re[c], im to out_im[c] (same fixed tree as the norm).
__global__ void __launch_bounds__(kThreads) k_chunk_inner(const double2 *__restrict__ a,
                                                          const double2 *__restrict__ b, uint64_t chunk,
                                                          double *__restrict__ out_re,
                                                          double *__restrict__ out_im)
{
    __shared__ double sh[32];
    const uint64_t base = (uint64_t)blockIdx.x * chunk;
    double re = 0.0, im = 0.0;
    for (uint64_t i = threadIdx.x; i < chunk; i += blockDim.x) {
        const double2 x = a[base + i], y = b[base + i];
        re = fma(x.x, y.x, fma(x.y, y.y, re));
        im = fma(x.x, y.y, fma(-x.y, y.x, im));
    }
    const double sr = block_sum(re, sh);
    const double si = block_sum(im, sh);
    if (threadIdx.x == 0) {
        out_re[blockIdx.x] = sr;
        out_im[blockIdx.x] = si;
    }
}

// Sum of the amplitudes themselves over chunks (the mean of Grover's diffusion
// 2|s><s| - I): block c writes re to out_re[c], im to
// out_im[c] (same fixed tree as the norm).
__global__ void __launch_bounds__(kThreads) k_chunk_sum(const double2 *__restrict__ a, uint64_t chunk,
                                                        double *__restrict__ out_re, double *__restrict__ out_im)
{
    __shared__ double sh[32];
    const uint64_t base = (uint64_t)blockIdx.x * chunk;
    double re = 0.0, im = 0.0;
    for (uint64_t i = threadIdx.x; i < chunk; i += blockDim.x) {
        const double2 x = a[base + i];
        re += x.x;
        im += x.y;
    }
    const double sr = block_sum(re, sh);
    const double si = block_sum(im, sh);
    if (threadIdx.x == 0) {
        out_re[blockIdx.x] = sr;
        out_im[blockIdx.x] = si;
    }
}

// alpha_i <- c - alpha_i for every amplitude (c = 2 mean: 2|s><s| - I).
__global__ void __launch_bounds__(kThreads) k_reflect(double2 *__restrict__ psi, uint64_t count, double2 c)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const double2 v = psi[i];
        psi[i] = make_double2(c.x - v.x, c.y - v.y);
    }
}

// Projection of a measured sub-register (R31): amplitudes whose masked bits
// equal val are scaled by s, every other one (all of them if zero_all) is 0.
__global__ void __launch_bounds__(kThreads) k_collapse(double2 *__restrict__ psi, uint64_t count, uint64_t mask,
                                                       uint64_t val, double s, int zero_all)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        if (zero_all || (i & mask) != val) {
            psi[i] = make_double2(0.0, 0.0);
        } else {
            const double2 v = psi[i];
            psi[i] = make_double2(v.x * s, v.y * s);
        }
    }
}

// Gaussian amplitudes (R19) generated on the device with the library's Philox.
__global__ void __launch_bounds__(kThreads) k_init_gaussian(double2 *__restrict__ psi, uint64_t count,
                                                            uint64_t gbase, uint64_t seed)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const u64x2 d = draw(seed, QSIM_TAG_GAUSS, gbase + i, 0);
        const double rad = sqrt(-2.0 * log(u01o(d.a)));
        double s, c;
        sincospi(2.0 * u01(d.b), &s, &c);
        psi[i] = make_double2(rad * c, rad * s);
    }
}

}  // namespace

static void sum_tree(Handle *h, const double *d_in, uint64_t count, double *d_out)
{
    prof_begin(h);
    k_sum_doubles<<<1, 1024, 0, h->stream>>>(d_in, count, count, d_out);
    prof_end(h, "k_sum_doubles", count * 8);
}

void launch_block_abs2(Handle *h, int blk_bits, double *d_out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const uint64_t chunk = 1ull << blk_bits;
    const uint64_t nb = h->local_dim() >> blk_bits;
    prof_begin(h);
    k_chunk_abs2<<<(unsigned)nb, kThreads, 0, h->stream>>>(h->psi, chunk, d_out);
    prof_end(h, "k_chunk_abs2", h->local_dim() * 16);
}

void launch_norm(Handle *h, double *d_out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    // chunks of 2^12 (or the whole shard if smaller), then one tree over them
    const int bb = h->nl < 12 ? h->nl : 12;
    const uint64_t nb = h->local_dim() >> bb;
    // d_out may live in the reduction workspace: keep it valid across a regrow
    const bool in_ws = h->d_red && d_out >= h->d_red && d_out < h->d_red + h->red_cap;
    const size_t off = in_ws ? (size_t)(d_out - h->d_red) : 0;
    ensure_red(h, nb + (nb >> 10) + 16);
    if (in_ws) d_out = h->d_red + off;
    launch_block_abs2(h, bb, h->d_red + 8);
    if (nb <= (1u << 20)) {
        sum_tree(h, h->d_red + 8, nb, d_out);
    } else {
        // two levels (n_local > 32)
        const uint64_t nb2 = nb >> 10;
        prof_begin(h);
        k_sum_doubles<<<(unsigned)nb2, 1024, 0, h->stream>>>(h->d_red + 8, 1024, 1024, h->d_red + 8 + nb);
        prof_end(h, "k_sum_doubles", nb * 8);
        sum_tree(h, h->d_red + 8 + nb, nb2, d_out);
    }
}

// tree sum of nb doubles at d_in (inside the reduction workspace, offset
// >= 8) into d_out; two levels above 2^20 partials
static void tree_sum_ws(Handle *h, const double *d_in, uint64_t nb, double *d_tmp, double *d_out)
{
    if (nb <= (1u << 20)) {
        sum_tree(h, d_in, nb, d_out);
        return;
    }
    const uint64_t nb2 = nb >> 10;
    prof_begin(h);
    k_sum_doubles<<<(unsigned)nb2, 1024, 0, h->stream>>>(d_in, 1024, 1024, d_tmp);
    prof_end(h, "k_sum_doubles", nb * 8);
    sum_tree(h, d_tmp, nb2, d_out);
}

void launch_inner(Handle *h, const double2 *a, const double2 *b, double *d_out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const int bb = h->nl < 12 ? h->nl : 12;
    const uint64_t nb = h->local_dim() >> bb;
    ensure_red(h, 2 * nb + (nb >> 9) + 16);
    double *re = h->d_red + 8, *im = re + nb, *tmp = im + nb;
    prof_begin(h);
    k_chunk_inner<<<(unsigned)nb, kThreads, 0, h->stream>>>(a, b, 1ull << bb, re, im);
    prof_end(h, "k_chunk_inner", h->local_dim() * 32);
    tree_sum_ws(h, re, nb, tmp, d_out);
    tree_sum_ws(h, im, nb, tmp, d_out + 1);
}

void launch_amp_sum(Handle *h, double *d_out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const int bb = h->nl < 12 ? h->nl : 12;
    const uint64_t nb = h->local_dim() >> bb;
    ensure_red(h, 2 * nb + (nb >> 9) + 16);
    double *re = h->d_red + 8, *im = re + nb, *tmp = im + nb;
    prof_begin(h);
    k_chunk_sum<<<(unsigned)nb, kThreads, 0, h->stream>>>(h->psi, 1ull << bb, re, im);
    prof_end(h, "k_chunk_sum", h->local_dim() * 16);
    tree_sum_ws(h, re, nb, tmp, d_out);
    tree_sum_ws(h, im, nb, tmp, d_out + 1);
}

void launch_reflect(Handle *h, double2 c)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const uint64_t count = h->local_dim();
    const uint64_t want = (count + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)h->num_sms * 8;
    prof_begin(h);
    k_reflect<<<(unsigned)(want < cap ? want : cap), kThreads, 0, h->stream>>>(h->psi, count, c);
    prof_end(h, "k_reflect", count * 32);
}

void launch_collapse(Handle *h, uint64_t mask, uint64_t val, double s, int zero_all)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const uint64_t count = h->local_dim();
    const uint64_t want = (count + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)h->num_sms * 8;
    prof_begin(h);
    k_collapse<<<(unsigned)(want < cap ? want : cap), kThreads, 0, h->stream>>>(h->psi, count, mask, val, s,
                                                                                 zero_all);
    // zeroed amplitudes are only written; the kept ones are read and written
    const uint64_t kept = zero_all ? 0 : count >> __builtin_popcountll(mask);
    prof_end(h, "k_collapse", count * 16 + kept * 16);
}

void launch_probs_contig(Handle *h, int pl, int m, double *d_out)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const uint64_t ny = 1ull << m;
    const uint64_t rest = h->local_dim() >> m;
    if (ny >= (uint64_t)h->num_sms * 64 && rest >= 64 && rest <= (1ull << 14)) {
        // many small marginal bins: a warp per bin (a block per bin spent its
        // time in scheduling: 5.97 TB/s on configs[3]'s 2^20 bins of 1024)
        const uint64_t want = (ny + 7) / 8;
        const uint64_t cap = (uint64_t)h->num_sms * 16;
        prof_begin(h);
        k_probs_warp<<<(unsigned)(want < cap ? want : cap), 256, 0, h->stream>>>(h->psi, pl, m, rest, ny, d_out);
        prof_end(h, "k_probs_warp", h->local_dim() * 16);
        return;
    }
    // chunks so that the grid has >= ~2 waves of blocks
    uint64_t nchunk = 1;
    while (ny * nchunk < (uint64_t)h->num_sms * 16 && rest / (nchunk * 2) >= kThreads && nchunk < 64) nchunk *= 2;
    const uint64_t chunk = rest / nchunk;
    ensure_red(h, ny * nchunk + 8);
    prof_begin(h);
    k_probs_contig<<<(unsigned)(ny * nchunk), kThreads, 0, h->stream>>>(h->psi, h->nl, pl, m, chunk,
                                                                         nchunk, h->d_red + 8);
    prof_end(h, "k_probs_contig", h->local_dim() * 16);
    prof_begin(h);
    k_probs_finish<<<(unsigned)((ny + 255) / 256), 256, 0, h->stream>>>(h->d_red + 8, ny, nchunk, d_out);
    prof_end(h, "k_probs_finish", ny * nchunk * 8);
}

void launch_init_gaussian(Handle *h, uint64_t seed)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    const uint64_t count = h->local_dim();
    const uint64_t gbase = (uint64_t)h->rank << h->nl;
    const uint64_t want = (count + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)h->num_sms * 8;
    prof_begin(h);
    k_init_gaussian<<<(unsigned)(want < cap ? want : cap), kThreads, 0, h->stream>>>(h->psi, count,
                                                                                      gbase, seed);
    prof_end(h, "k_init_gaussian", count * 16);
}

}  // namespace qs
