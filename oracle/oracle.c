/*
 * oracle.c -- the CPU ORACLE for the Niwa-Matsumoto-Imai state-vector simulator.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (the sm_100a library
 * libqsim.so and its Python binding) may include, link, import or execute this
 * file.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it.  It shares no code, header, table or constant
 * generator with the CUDA path: the counter-based RNG, the gate matrices, the
 * circuits of BASELINE.json configs[0..4] and every reduction are written out
 * here a second time, independently, from the paper and from the
 * readings listed in DESIGN.md §3.
 *
 * Style: plain, slow, obviously correct.  Every kernel is the paper's in-place
 * pair loop (§2.2.1) written literally; the only
 * parallelism is an OpenMP `parallel for` over independent pairs, the paper's
 * own SMP decomposition, which is bit-identical for any
 * thread count because each pair's arithmetic is independent.
 * Complex numbers are C99 `double complex` (fp64).
 *
 * Qubit convention: qubit 0 is the MSB; qubit q of an n-qubit
 * register is bit (n-1-q) of the basis index, stride 2^(n-1-q).
 *
 * Parity status of each function is listed in DESIGN.md §4 ("pins").
 */
#include <complex.h>
#include <omp.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------------ */
/* Counter-based RNG: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).     */
/* Contract: DESIGN.md §3 reading R1.  The paper is silent on its RNG        */
/* ("Each experiment uses different initial random seed") */
/* ------------------------------------------------------------------------ */

enum { TAG_GATE = 1, TAG_HAAR = 2, TAG_PAIR = 3, TAG_OPNOISE = 4, TAG_MARK = 5,
       TAG_BASE = 6, TAG_GAUSS = 7, TAG_PAULI = 8, TAG_MEASURE = 9, TAG_SHOR = 10 };

/* One Philox4x32 round: two 32x32->64 multiplies, xor with key. */
static void philox_round(uint32_t c[4], const uint32_t k[2])
{
    const uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

/* Raw Philox4x32-10 block: 10 rounds, key bumped by the Weyl constants
 * between rounds. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c[4] = { ctr[0], ctr[1], ctr[2], ctr[3] };
    uint32_t k[2] = { key[0], key[1] };
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* draw(seed, tag, i, j) -> (a, b): key = (seed lo, seed hi),
 * counter = (i lo, i hi, j, tag); a = x0 | x1<<32, b = x2 | x3<<32. */
void orc_draw(uint64_t seed, uint32_t tag, uint64_t i, uint32_t j, uint64_t ab[2])
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t ctr[4] = { (uint32_t)i, (uint32_t)(i >> 32), j, tag };
    uint32_t x[4];
    orc_philox4x32_10(ctr, key, x);
    ab[0] = (uint64_t)x[0] | ((uint64_t)x[1] << 32);
    ab[1] = (uint64_t)x[2] | ((uint64_t)x[3] << 32);
}

/* u01(a) in [0,1): top 53 bits. */
double orc_u01(uint64_t a) { return (double)(a >> 11) * 0x1p-53; }
/* u01o(a) in (0,1]: used under the logarithm of Box-Muller. */
double orc_u01o(uint64_t a) { return (double)((a >> 11) + 1) * 0x1p-53; }
/* uint(a, m) = floor(a*m / 2^64), an integer in [0, m). */
uint64_t orc_uint(uint64_t a, uint64_t m)
{
    return (uint64_t)(((unsigned __int128)a * (unsigned __int128)m) >> 64);
}
/* Standard normal, Box-Muller cos branch. */
double orc_normal(uint64_t seed, uint32_t tag, uint64_t i, uint32_t j)
{
    uint64_t ab[2];
    orc_draw(seed, tag, i, j, ab);
    return sqrt(-2.0 * log(orc_u01o(ab[0]))) * cos(2.0 * ORC_PI * orc_u01(ab[1]));
}

/* ------------------------------------------------------------------------ */
/* Gate matrices.  U = (u11 u12; u21 u22) stored row-major [u11,u12,u21,u22] */
/* (PAPER.md:129-135).                                                        */
/* ------------------------------------------------------------------------ */

static void mat_mul(const cplx A[4], const cplx B[4], cplx C[4])
{
    cplx r[4];
    r[0] = A[0] * B[0] + A[1] * B[2];
    r[1] = A[0] * B[1] + A[1] * B[3];
    r[2] = A[2] * B[0] + A[3] * B[2];
    r[3] = A[2] * B[1] + A[3] * B[3];
    memcpy(C, r, sizeof r);
}

/* Rotation U_R(theta) = (cos -sin; sin cos)          PAPER.md:542-547 (§3.2) */
void orc_mat_ur(double theta, cplx U[4])
{
    U[0] = cos(theta); U[1] = -sin(theta); U[2] = sin(theta); U[3] = cos(theta);
}
/* Phase shift U_P1(phi) = diag(1, e^{i phi}) */
void orc_mat_up1(double phi, cplx U[4])
{
    U[0] = 1.0; U[1] = 0.0; U[2] = 0.0; U[3] = cos(phi) + I * sin(phi);
}
/* Phase shift U_P2(phi) = diag(e^{i phi}, 1) */
void orc_mat_up2(double phi, cplx U[4])
{
    U[0] = cos(phi) + I * sin(phi); U[1] = 0.0; U[2] = 0.0; U[3] = 1.0;
}

/* Angle-form gate kinds (reading R12-R14):
 *   ORC_RP   : U_R(a0) . U_P1(a1)          H = RP(pi/4, pi), NOT = RP(pi/2, pi)
 *              (PAPER.md:563-566 read as matrix products)
 *   ORC_P1   : U_P1(a0)                    R_d = P1(pi/2^d)
 *   ORC_HAAR : U_P2(a0) U_P1(a1) U_R(a2) U_P1(a3)   general 1q gate (R12)      */
enum { ORC_RP = 0, ORC_P1 = 1, ORC_HAAR = 2 };

int orc_kind_nangles(int kind) { return kind == ORC_RP ? 2 : kind == ORC_P1 ? 1 : 4; }

void orc_mat_angles(int kind, const double *ang, cplx U[4])
{
    cplx A[4], B[4], C[4];
    if (kind == ORC_RP) {
        orc_mat_ur(ang[0], A); orc_mat_up1(ang[1], B); mat_mul(A, B, U);
    } else if (kind == ORC_P1) {
        orc_mat_up1(ang[0], U);
    } else {
        orc_mat_up2(ang[0], A); orc_mat_up1(ang[1], B); mat_mul(A, B, C);
        orc_mat_ur(ang[2], A); mat_mul(C, A, B);
        orc_mat_up1(ang[3], A); mat_mul(B, A, U);
    }
}

/* Operational error (§3.2): each angle of angle-form gate
 * number g gets an independent Gaussian deviation sigma * z, z drawn from
 * counter (seed, OPNOISE, g, slot) -- fresh per application (R15). */
void orc_mat_angles_noisy(int kind, const double *ang, uint64_t seed, double sigma,
                          uint64_t g, cplx U[4])
{
    double a[4];
    int na = orc_kind_nangles(kind);
    for (int s = 0; s < na; ++s)
        a[s] = ang[s] + (sigma != 0.0 ? sigma * orc_normal(seed, TAG_OPNOISE, g, (uint32_t)s) : 0.0);
    orc_mat_angles(kind, a, U);
}

/* Haar-random angles for gate index i (R12): xi = u01(a0), theta = acos(sqrt(xi)),
 * alpha = 2pi u01(b0), beta = 2pi u01(a1), gamma = 2pi u01(b1).
 * Returned in ORC_HAAR slot order (alpha, beta, theta, gamma). */
void orc_haar_angles(uint64_t seed, uint64_t i, double ang[4])
{
    uint64_t d0[2], d1[2];
    orc_draw(seed, TAG_HAAR, i, 0, d0);
    orc_draw(seed, TAG_HAAR, i, 1, d1);
    ang[0] = 2.0 * ORC_PI * orc_u01(d0[1]);
    ang[1] = 2.0 * ORC_PI * orc_u01(d1[0]);
    ang[2] = acos(sqrt(orc_u01(d0[0])));
    ang[3] = 2.0 * ORC_PI * orc_u01(d1[1]);
}

/* ------------------------------------------------------------------------ */
/* Evolution kernels (§2.2)                                         */
/* ------------------------------------------------------------------------ */

/* Index mask of a set of qubits given as a bit set over qubit numbers. */
static uint64_t qubits_to_index_mask(int n, uint64_t qmask)
{
    uint64_t m = 0;
    for (int q = 0; q < n; ++q)
        if ((qmask >> q) & 1u) m |= (uint64_t)1 << (n - 1 - q);
    return m;
}

/* Single-qubit gate U on qubit q, in place:
 * rows j and j + 2^(n-q-1) are paired; the new j-th element is kept in a
 * temporary t1 while the partner is written, then t1 is stored. */
void orc_apply_1q(cplx *psi, int n, int q, const cplx U[4])
{
    const uint64_t dim = (uint64_t)1 << n;
    const uint64_t s = (uint64_t)1 << (n - 1 - q);
    #pragma omp parallel for schedule(static) if (dim >= (1u << 16))
    for (int64_t jj = 0; jj < (int64_t)dim; ++jj) {
        uint64_t j = (uint64_t)jj;
        if (j & s) continue;
        cplx x = psi[j], y = psi[j + s];
        cplx t1 = x * U[0] + y * U[1];
        psi[j + s] = x * U[2] + y * U[3];
        psi[j] = t1;
    }
}

/* Controlled gate: CTX[j] = X[j] where the control bits of
 * j match, I[j] otherwise; "in many controlled bit cases, it is easy to
 * extend" -> ctrl_mask is a set of qubits, ctrl_vals their required values. */
void orc_apply_ctrl(cplx *psi, int n, uint64_t ctrl_mask, uint64_t ctrl_vals, int q,
                    const cplx U[4])
{
    const uint64_t dim = (uint64_t)1 << n;
    const uint64_t s = (uint64_t)1 << (n - 1 - q);
    const uint64_t cm = qubits_to_index_mask(n, ctrl_mask);
    const uint64_t cv = qubits_to_index_mask(n, ctrl_vals & ctrl_mask);
    #pragma omp parallel for schedule(static) if (dim >= (1u << 16))
    for (int64_t jj = 0; jj < (int64_t)dim; ++jj) {
        uint64_t j = (uint64_t)jj;
        if (j & s) continue;
        if ((j & cm) != cv) continue;
        cplx x = psi[j], y = psi[j + s];
        cplx t1 = x * U[0] + y * U[1];
        psi[j + s] = x * U[2] + y * U[3];
        psi[j] = t1;
    }
}

/* SWAP of qubits q1, q2: exchange the amplitudes of |..b1..b2..> and
 * |..b2..b1..> (the final swaps of the QFT, reading R7). */
void orc_swap(cplx *psi, int n, int q1, int q2)
{
    if (q1 == q2) return;
    const uint64_t dim = (uint64_t)1 << n;
    const uint64_t s1 = (uint64_t)1 << (n - 1 - q1), s2 = (uint64_t)1 << (n - 1 - q2);
    #pragma omp parallel for schedule(static) if (dim >= (1u << 16))
    for (int64_t jj = 0; jj < (int64_t)dim; ++jj) {
        uint64_t j = (uint64_t)jj;
        if ((j & s1) && !(j & s2)) {
            uint64_t k = (j ^ s1) | s2;
            cplx t = psi[j]; psi[j] = psi[k]; psi[k] = t;
        }
    }
}

/* Sign-changing operator V_f for f = delta_{x,idx} (§5.3),
 * in its ancilla-free phase-flip form (reading R17). */
void orc_phase_flip(cplx *psi, int n, uint64_t idx)
{
    (void)n;
    psi[idx] = -psi[idx];
}

/* Pauli matrices of the depolarizing channel (§3.1). */
void orc_pauli(int which, cplx U[4])
{
    if (which == 1) { U[0] = 0; U[1] = 1; U[2] = 1; U[3] = 0; }          /* sigma_x */
    else if (which == 2) { U[0] = 0; U[1] = -I; U[2] = I; U[3] = 0; }    /* sigma_y */
    else { U[0] = 1; U[1] = 0; U[2] = 0; U[3] = -1; }                   /* sigma_z */
}

/* ------------------------------------------------------------------------ */
/* Reductions                                                                 */
/* ------------------------------------------------------------------------ */

/* Pairwise (recursive halving) sum of |psi_j|^2 over [lo, lo+len)   (R23). */
static double pairwise_abs2(const cplx *psi, uint64_t lo, uint64_t len)
{
    if (len <= 8) {
        double s = 0.0;
        for (uint64_t j = lo; j < lo + len; ++j)
            s += creal(psi[j]) * creal(psi[j]) + cimag(psi[j]) * cimag(psi[j]);
        return s;
    }
    uint64_t h = len / 2;
    return pairwise_abs2(psi, lo, h) + pairwise_abs2(psi, lo + h, len - h);
}

/* Sum_i |alpha_i|^2 (§2.1). */
double orc_norm(const cplx *psi, int n)
{
    const uint64_t dim = (uint64_t)1 << n;
    if (dim < (1u << 20)) return pairwise_abs2(psi, 0, dim);
    /* same pairwise tree, top levels computed in parallel */
    const int top = 10;
    const uint64_t nb = (uint64_t)1 << top, bl = dim >> top;
    double part[1 << 10];
    #pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < (int64_t)nb; ++b) part[b] = pairwise_abs2(psi, (uint64_t)b * bl, bl);
    for (uint64_t w = nb; w > 1; w >>= 1)
        for (uint64_t b = 0; b < w / 2; ++b) part[b] = part[2 * b] + part[2 * b + 1];
    return part[0];
}

/* Marginal probabilities of the sub-register of qubits [lo, lo+m) (qubit lo is
 * its MSB): P(y) = sum of |alpha_j|^2 over j whose sub-register value is y.
 * Each P(y) is a pairwise sum over its 2^(n-m) members. */
void orc_probs(const cplx *psi, int n, int lo, int m, double *out)
{
    const uint64_t ny = (uint64_t)1 << m;
    const int shift = n - lo - m;
    const uint64_t nrest = (uint64_t)1 << (n - m);
    #pragma omp parallel for schedule(static)
    for (int64_t yy = 0; yy < (int64_t)ny; ++yy) {
        uint64_t y = (uint64_t)yy;
        double *tmp = (double *)malloc(sizeof(double) * nrest);
        for (uint64_t r = 0; r < nrest; ++r) {
            uint64_t low = r & (((uint64_t)1 << shift) - 1);
            uint64_t high = r >> shift;
            uint64_t j = (high << (shift + m)) | (y << shift) | low;
            tmp[r] = creal(psi[j]) * creal(psi[j]) + cimag(psi[j]) * cimag(psi[j]);
        }
        uint64_t w = nrest;
        while (w > 1) {
            uint64_t h = w / 2;
            for (uint64_t k = 0; k < h; ++k) tmp[k] = tmp[2 * k] + tmp[2 * k + 1];
            if (w & 1) { tmp[h] = tmp[w - 1]; w = h + 1; } else w = h;
        }
        out[y] = tmp[0];
        free(tmp);
    }
}

/* Measurement (§2.2.3): given r in [0,1), the integer i with
 * sum_{j<i} |a_j|^2 <= r < sum_{j<=i} |a_j|^2, by a sequential scan.  If
 * rounding leaves r >= the total, the largest i with a_i != 0 (reading R21). */
uint64_t orc_measure(const cplx *psi, int n, double r)
{
    const uint64_t dim = (uint64_t)1 << n;
    double acc = 0.0;
    uint64_t last_nz = 0;
    for (uint64_t i = 0; i < dim; ++i) {
        double p = creal(psi[i]) * creal(psi[i]) + cimag(psi[i]) * cimag(psi[i]);
        if (p != 0.0) last_nz = i;
        acc += p;
        if (r < acc) return i;
    }
    return last_nz;
}

/* Measurement of the sub-register of qubits [lo, lo+m) (PAPER.md:391-404
 * applied to the marginal distribution; reading R31): y = the smallest value
 * with sum_{y'<=y} P(y') > r, scanning P in order (P from orc_probs); if
 * rounding leaves r >= the total, the largest y with P(y) > 0.  With collapse
 * != 0 the state is projected onto that value and renormalised:
 * alpha_j <- alpha_j / sqrt(P(y)) where the sub-register of j equals y, 0
 * elsewhere. */
uint64_t orc_measure_range(cplx *psi, int n, int lo, int m, double r, int collapse)
{
    const uint64_t ny = (uint64_t)1 << m;
    double *P = (double *)malloc(sizeof(double) * ny);
    orc_probs(psi, n, lo, m, P);
    double acc = 0.0;
    uint64_t y = ny, last_nz = 0;
    for (uint64_t v = 0; v < ny; ++v) {
        if (P[v] > 0.0) last_nz = v;
        acc += P[v];
        if (r < acc) { y = v; break; }
    }
    if (y == ny) y = last_nz;
    if (collapse) {
        const double s = 1.0 / sqrt(P[y]);
        const uint64_t dim = (uint64_t)1 << n;
        const int shift = n - lo - m;
        #pragma omp parallel for schedule(static)
        for (int64_t jj = 0; jj < (int64_t)dim; ++jj) {
            uint64_t j = (uint64_t)jj;
            if (((j >> shift) & (ny - 1)) == y) psi[j] *= s;
            else psi[j] = 0.0;
        }
    }
    free(P);
    return y;
}

/* Pairwise sum of conj(a_j) b_j over [lo, lo+len) (R23). */
static cplx pairwise_inner(const cplx *a, const cplx *b, uint64_t lo, uint64_t len)
{
    if (len <= 8) {
        cplx s = 0.0;
        for (uint64_t j = lo; j < lo + len; ++j) s += conj(a[j]) * b[j];
        return s;
    }
    uint64_t h = len / 2;
    return pairwise_inner(a, b, lo, h) + pairwise_inner(a, b, lo + h, len - h);
}

/* Inner product <a|b> = sum_j conj(a_j) b_j; the paper's fidelity is its
 * modulus, "the inner product of the correct state and the simulated state"
 * (reading C26/R32). */
void orc_inner(const cplx *a, const cplx *b, int n, cplx *out)
{
    *out = pairwise_inner(a, b, 0, (uint64_t)1 << n);
}

/* ------------------------------------------------------------------------ */
/* Basis permutations: modular multiplication / exponentiation               */
/* (§2.3.3; applied semantically as a permutation, R9/R10) */
/* ------------------------------------------------------------------------ */

/* Out-of-place controlled modular multiplication on the work register of
 * qubits [wlo, wlo+wm): v -> v*c mod N if v < N and the control qubits
 * match, identity otherwise (R10).  Each index has exactly one destination. */
void orc_modmul(cplx *psi, int n, int wlo, int wm, uint64_t ctrl_mask, uint64_t ctrl_vals,
                uint64_t c, uint64_t N)
{
    const uint64_t dim = (uint64_t)1 << n;
    const int shift = n - wlo - wm;
    const uint64_t vmask = (((uint64_t)1 << wm) - 1) << shift;
    const uint64_t cm = qubits_to_index_mask(n, ctrl_mask);
    const uint64_t cv = qubits_to_index_mask(n, ctrl_vals & ctrl_mask);
    cplx *out = (cplx *)malloc(sizeof(cplx) * dim);
    #pragma omp parallel for schedule(static) if (dim >= (1u << 16))
    for (int64_t jj = 0; jj < (int64_t)dim; ++jj) {
        uint64_t j = (uint64_t)jj;
        uint64_t v = (j & vmask) >> shift;
        uint64_t dst = j;
        if ((j & cm) == cv && v < N) {
            uint64_t w = (uint64_t)(((unsigned __int128)v * c) % N);
            dst = (j & ~vmask) | (w << shift);
        }
        out[dst] = psi[j];
    }
    memcpy(psi, out, sizeof(cplx) * dim);
    free(out);
}

/* a^e mod N by repeated squaring (classical, PAPER.md:502-509 footnote). */
uint64_t orc_powmod(uint64_t a, uint64_t e, uint64_t N)
{
    unsigned __int128 r = 1 % N, b = a % N;
    while (e) {
        if (e & 1) r = (r * b) % N;
        b = (b * b) % N;
        e >>= 1;
    }
    return (uint64_t)r;
}

uint64_t orc_gcd(uint64_t a, uint64_t b)
{
    while (b) { uint64_t t = a % b; a = b; b = t; }
    return a;
}

/* ------------------------------------------------------------------------ */
/* Circuits (§2.3)                                                  */
/* ------------------------------------------------------------------------ */

/* Noise context shared by the angle-form gates of one circuit. */
typedef struct {
    uint64_t seed;   /* OPNOISE seed */
    double sigma;    /* 0 -> noiseless */
    uint64_t g;      /* angle-form gate counter, in circuit order (R15) */
} orc_noise_t;

/* Apply one angle-form gate (optionally controlled); advances g. */
void orc_apply_angles(cplx *psi, int n, orc_noise_t *nz, int kind, const double *ang,
                      uint64_t ctrl_mask, uint64_t ctrl_vals, int q)
{
    cplx U[4];
    orc_mat_angles_noisy(kind, ang, nz->seed, nz->sigma, nz->g, U);
    nz->g += 1;
    if (ctrl_mask) orc_apply_ctrl(psi, n, ctrl_mask, ctrl_vals, q, U);
    else orc_apply_1q(psi, n, q, U);
}

/* QFT circuit on qubits [lo, lo+m) (§2.3.2; readings R6-R8):
 *   for j = 0..m-1: H(lo+j); for k = j+1..m-1: R_{k-j} controlled by lo+k on lo+j
 *   then SWAP(lo+j, lo+m-1-j), j < m/2.
 * R_d = diag(1, e^{+-i pi / 2^d}); inverse = same order, negated phases.
 * Noiseless gates are the constant matrices (H with 1/sqrt2 = M_SQRT1_2);
 * when nz->sigma > 0 every H is RP(pi/4 + x, pi + y) and every R_d is
 * P1(+-pi/2^d + x).  g advances per H and per
 * R_d either way; swaps are noiseless (R14). */
void orc_qft(cplx *psi, int n, int lo, int m, int inverse, orc_noise_t *nz)
{
    const double sgn = inverse ? -1.0 : 1.0;
    const double r = 0.70710678118654752440; /* M_SQRT1_2 */
    cplx H[4] = { r, r, r, -r };
    for (int j = 0; j < m; ++j) {
        if (nz->sigma > 0.0) {
            double ang[2] = { ORC_PI / 4.0, ORC_PI };
            orc_apply_angles(psi, n, nz, ORC_RP, ang, 0, 0, lo + j);
        } else {
            orc_apply_1q(psi, n, lo + j, H);
            nz->g += 1;
        }
        for (int k = j + 1; k < m; ++k) {
            double phi = sgn * ORC_PI / ldexp(1.0, k - j);
            uint64_t cm = (uint64_t)1 << (lo + k);
            if (nz->sigma > 0.0) {
                orc_apply_angles(psi, n, nz, ORC_P1, &phi, cm, cm, lo + j);
            } else {
                cplx R[4] = { 1.0, 0.0, 0.0, cos(phi) + I * sin(phi) };
                orc_apply_ctrl(psi, n, cm, cm, lo + j, R);
                nz->g += 1;
            }
        }
    }
    for (int j = 0; j < m / 2; ++j) orc_swap(psi, n, lo + j, lo + m - 1 - j);
}

/* Approximate QFT (§2.3.2: "the controlled phase shift
 * gates acting on distantly separated qubits contribute only exponentially
 * small phases"; Barenco et al.): the circuit of orc_qft with every R_d of
 * distance d = k - j > b left out (reading R30).  b >= m-1 is the exact QFT.
 * The gate counter g advances only for gates that are applied. */
void orc_aqft(cplx *psi, int n, int lo, int m, int b, int inverse, orc_noise_t *nz)
{
    const double sgn = inverse ? -1.0 : 1.0;
    const double r = 0.70710678118654752440; /* M_SQRT1_2 */
    cplx H[4] = { r, r, r, -r };
    for (int j = 0; j < m; ++j) {
        if (nz->sigma > 0.0) {
            double ang[2] = { ORC_PI / 4.0, ORC_PI };
            orc_apply_angles(psi, n, nz, ORC_RP, ang, 0, 0, lo + j);
        } else {
            orc_apply_1q(psi, n, lo + j, H);
            nz->g += 1;
        }
        for (int k = j + 1; k < m; ++k) {
            if (k - j > b) continue;
            double phi = sgn * ORC_PI / ldexp(1.0, k - j);
            uint64_t cm = (uint64_t)1 << (lo + k);
            if (nz->sigma > 0.0) {
                orc_apply_angles(psi, n, nz, ORC_P1, &phi, cm, cm, lo + j);
            } else {
                cplx R[4] = { 1.0, 0.0, 0.0, cos(phi) + I * sin(phi) };
                orc_apply_ctrl(psi, n, cm, cm, lo + j, R);
                nz->g += 1;
            }
        }
    }
    for (int j = 0; j < m / 2; ++j) orc_swap(psi, n, lo + j, lo + m - 1 - j);
}

/* Hadamard transform H_n on qubits [lo, lo+m) with the constant H
 * (§2.3.1). */
void orc_hadamard_range(cplx *psi, int n, int lo, int m)
{
    const double r = 0.70710678118654752440;
    cplx H[4] = { r, r, r, -r };
    for (int q = lo; q < lo + m; ++q) orc_apply_1q(psi, n, q, H);
}

/* Definition of the DFT output: beta_x = 2^{-n/2}
 * sum_y w^{+-xy} alpha_y, w = e^{2 pi i / 2^n}; used to check sampled
 * outputs at sizes where the circuit is too slow on the CPU.  x*y is reduced
 * mod 2^n exactly in integers; w^t is taken from two exact-to-1ulp tables. */
void orc_dft_samples(const cplx *psi, int n, int inverse, const uint64_t *xs, int nx, cplx *out)
{
    const uint64_t dim = (uint64_t)1 << n;
    const int hb = n / 2, lb = n - hb;
    const uint64_t nh = (uint64_t)1 << hb, nl = (uint64_t)1 << lb;
    cplx *th = (cplx *)malloc(sizeof(cplx) * nh), *tl = (cplx *)malloc(sizeof(cplx) * nl);
    const double sgn = inverse ? -1.0 : 1.0;
    for (uint64_t t = 0; t < nh; ++t) {
        double ph = sgn * 2.0 * ORC_PI * (double)(t << lb) / (double)dim;
        th[t] = cos(ph) + I * sin(ph);
    }
    for (uint64_t t = 0; t < nl; ++t) {
        double ph = sgn * 2.0 * ORC_PI * (double)t / (double)dim;
        tl[t] = cos(ph) + I * sin(ph);
    }
    const double scale = 1.0 / sqrt((double)dim);
    for (int s = 0; s < nx; ++s) {
        const uint64_t x = xs[s];
        /* pairwise over 2^10 partial sums for accuracy */
        const int top = n > 10 ? 10 : n;
        const uint64_t nb = (uint64_t)1 << top, bl = dim >> top;
        cplx *part = (cplx *)malloc(sizeof(cplx) * nb);
        #pragma omp parallel for schedule(static)
        for (int64_t b = 0; b < (int64_t)nb; ++b) {
            cplx acc = 0.0;
            for (uint64_t y = (uint64_t)b * bl; y < (uint64_t)(b + 1) * bl; ++y) {
                uint64_t t = (x * y) & (dim - 1);
                acc += th[t >> lb] * tl[t & (nl - 1)] * psi[y];
            }
            part[b] = acc;
        }
        for (uint64_t w = nb; w > 1; w >>= 1)
            for (uint64_t b = 0; b < w / 2; ++b) part[b] = part[2 * b] + part[2 * b + 1];
        out[s] = part[0] * scale;
        free(part);
    }
    free(th); free(tl);
}

/* ------------------------------------------------------------------------ */
/* BASELINE.json configs[0..4], oracle recipes (R16-R20)        */
/* ------------------------------------------------------------------------ */

/* configs[0]: random circuit on |0..0>, ngates gates from `seed`: with
 * p = 0.7 a Haar-random 2x2 on a uniform qubit, else a CNOT on a uniform
 * ordered pair (R17).  kinds_out (optional) receives 0 = Haar, 1 = CNOT;
 * q_out receives (target, control) per gate (control = -1 for Haar). */
void orc_cfg0(cplx *psi, int n, uint64_t seed, int ngates, int *kinds_out, int *q_out)
{
    const uint64_t dim = (uint64_t)1 << n;
    memset(psi, 0, sizeof(cplx) * dim);
    psi[0] = 1.0;
    orc_noise_t nz = { seed, 0.0, 0 };
    for (int g = 0; g < ngates; ++g) {
        uint64_t d[2];
        orc_draw(seed, TAG_GATE, (uint64_t)g, 0, d);
        if (orc_u01(d[0]) < 0.7) {
            int q = (int)orc_uint(d[1], (uint64_t)n);
            double ang[4];
            orc_haar_angles(seed, (uint64_t)g, ang);
            orc_apply_angles(psi, n, &nz, ORC_HAAR, ang, 0, 0, q);
            if (kinds_out) kinds_out[g] = 0;
            if (q_out) { q_out[2 * g] = q; q_out[2 * g + 1] = -1; }
        } else {
            uint64_t e[2];
            orc_draw(seed, TAG_PAIR, (uint64_t)g, 0, e);
            int c = (int)orc_uint(e[0], (uint64_t)n);
            int t = (int)orc_uint(e[1], (uint64_t)(n - 1));
            if (t >= c) t += 1;
            cplx X[4] = { 0.0, 1.0, 1.0, 0.0 };
            orc_apply_ctrl(psi, n, (uint64_t)1 << c, (uint64_t)1 << c, t, X);
            if (kinds_out) kinds_out[g] = 1;
            if (q_out) { q_out[2 * g] = t; q_out[2 * g + 1] = c; }
        }
    }
}

/* Marked index of configs[1] (R20). */
uint64_t orc_grover_mark(uint64_t seed, int n)
{
    uint64_t d[2];
    orc_draw(seed, TAG_MARK, 0, 0, d);
    return orc_uint(d[0], (uint64_t)1 << n);
}

/* One G-iteration -H_n V_{f0} H_n V_{fk}, literally (§5.3). */
void orc_grover_iteration(cplx *psi, int n, uint64_t k)
{
    const uint64_t dim = (uint64_t)1 << n;
    orc_phase_flip(psi, n, k);
    orc_hadamard_range(psi, n, 0, n);
    orc_phase_flip(psi, n, 0);
    orc_hadamard_range(psi, n, 0, n);
    for (uint64_t j = 0; j < dim; ++j) psi[j] = -psi[j];
}

/* configs[1]: H_n|0>, then `iters` G-iterations, trace[t] = |alpha_k|^2 after
 * iteration t+1. */
void orc_cfg1(cplx *psi, int n, uint64_t seed, int iters, double *trace)
{
    const uint64_t dim = (uint64_t)1 << n;
    memset(psi, 0, sizeof(cplx) * dim);
    psi[0] = 1.0;
    orc_hadamard_range(psi, n, 0, n);
    uint64_t k = orc_grover_mark(seed, n);
    for (int t = 0; t < iters; ++t) {
        orc_grover_iteration(psi, n, k);
        if (trace) trace[t] = creal(psi[k]) * creal(psi[k]) + cimag(psi[k]) * cimag(psi[k]);
    }
}

/* configs[2] input (R19): alpha_idx = complex Gaussian from draw(seed, GAUSS,
 * idx, 0) (Box-Muller, re = cos branch, im = sin branch), then divided by
 * sqrt(pairwise sum |alpha|^2). */
void orc_gaussian_state(cplx *psi, int n, uint64_t seed)
{
    const uint64_t dim = (uint64_t)1 << n;
    #pragma omp parallel for schedule(static)
    for (int64_t jj = 0; jj < (int64_t)dim; ++jj) {
        uint64_t d[2];
        orc_draw(seed, TAG_GAUSS, (uint64_t)jj, 0, d);
        double rad = sqrt(-2.0 * log(orc_u01o(d[0])));
        double ph = 2.0 * ORC_PI * orc_u01(d[1]);
        psi[jj] = rad * cos(ph) + I * (rad * sin(ph));
    }
    double s = orc_norm(psi, n);
    double inv = 1.0 / sqrt(s);
    #pragma omp parallel for schedule(static)
    for (int64_t jj = 0; jj < (int64_t)dim; ++jj) psi[jj] *= inv;
}

/* configs[2]: Gaussian input, then the QFT circuit on all n qubits. */
void orc_cfg2(cplx *psi, int n, uint64_t seed)
{
    orc_gaussian_state(psi, n, seed);
    orc_noise_t nz = { seed, 0.0, 0 };
    orc_qft(psi, n, 0, n, 0, &nz);
}

/* Base of configs[3] (R11): a_t = 2 + uint(draw(seed, BASE, t, 0).a, N-3),
 * first with gcd(a_t, N) = 1. */
uint64_t orc_shor_base(uint64_t seed, uint64_t N)
{
    for (uint64_t t = 0;; ++t) {
        uint64_t d[2];
        orc_draw(seed, TAG_BASE, t, 0, d);
        uint64_t a = 2 + orc_uint(d[0], N - 3);
        if (orc_gcd(a, N) == 1) return a;
    }
}

/* configs[3] (order finding, §5.1, readings R8-R11):
 * exponent register = qubits [0, ne), work register = qubits [ne, ne+nw),
 * start |e=0>|w=1>, H on every exponent qubit (angle form when sigma > 0),
 * for j = 0..ne-1 the modular multiplication by a^(2^j) mod N controlled on
 * exponent bit j (= qubit ne-1-j), inverse QFT on the exponent register,
 * probs_out[e] = sum_w |psi(e, w)|^2.  psi must hold 2^(ne+nw) amplitudes. */
void orc_cfg3(cplx *psi, int ne, int nw, uint64_t N, uint64_t a, uint64_t seed, double sigma,
              double *probs_out)
{
    const int n = ne + nw;
    const uint64_t dim = (uint64_t)1 << n;
    memset(psi, 0, sizeof(cplx) * dim);
    psi[1] = 1.0;                                   /* e = 0, w = 1 */
    orc_noise_t nz = { seed, sigma, 0 };
    const double r = 0.70710678118654752440;
    cplx H[4] = { r, r, r, -r };
    for (int q = 0; q < ne; ++q) {
        if (sigma > 0.0) {
            double ang[2] = { ORC_PI / 4.0, ORC_PI };
            orc_apply_angles(psi, n, &nz, ORC_RP, ang, 0, 0, q);
        } else {
            orc_apply_1q(psi, n, q, H);
            nz.g += 1;
        }
    }
    for (int j = 0; j < ne; ++j) {
        uint64_t c = orc_powmod(a, (uint64_t)1 << j, N);
        uint64_t cm = (uint64_t)1 << (ne - 1 - j);
        orc_modmul(psi, n, ne, nw, cm, cm, c, N);
    }
    orc_qft(psi, n, 0, ne, 1, &nz);
    if (probs_out) orc_probs(psi, n, 0, ne, probs_out);
}

/* Depolarizing channel on pure-state trajectories (§3.1;
 * reading R16): for each qubit q in qmask, u = u01(draw(seed, PAULI, epoch, q).a);
 * u < p/3 -> sigma_x, u < 2p/3 -> sigma_y, u < p -> sigma_z, else identity.
 * Events are appended as (epoch, q, pauli) triples into ev[*nev..cap). */
void orc_inject_paulis(cplx *psi, int n, uint64_t seed, uint64_t epoch, uint64_t qmask,
                       double p, int *ev, int cap, int *nev)
{
    for (int q = 0; q < n; ++q) {
        if (!((qmask >> q) & 1u)) continue;
        uint64_t d[2];
        orc_draw(seed, TAG_PAULI, epoch, (uint32_t)q, d);
        double u = orc_u01(d[0]);
        int which = u < p / 3.0 ? 1 : u < 2.0 * p / 3.0 ? 2 : u < p ? 3 : 0;
        if (!which) continue;
        cplx P[4];
        orc_pauli(which, P);
        orc_apply_1q(psi, n, q, P);
        if (ev && *nev < cap) {
            ev[3 * *nev] = (int)epoch; ev[3 * *nev + 1] = q; ev[3 * *nev + 2] = which;
        }
        *nev += 1;
    }
}

/* configs[4] (noisy brickwork, reading R18): `layers` layers, each:
 * n Haar gates (qubit 0..n-1, HAAR index l*n+q) with angle noise sigma,
 * CNOTs on (2k, 2k+1) for even l / (2k+1, 2k+2) for odd l, control = lower
 * qubit, NOT = RP(pi/2, pi) with angle noise, then a depolarizing injection
 * on every qubit: u = u01(draw(seed, PAULI, l, q).a),
 * u < p/3 -> X, < 2p/3 -> Y, < p -> Z.  Events are written as triples
 * (layer, qubit, pauli 1..3) into ev (capacity cap); returns the count. */
int orc_cfg4(cplx *psi, int n, int layers, uint64_t seed, double sigma, double p,
             int *ev, int cap)
{
    const uint64_t dim = (uint64_t)1 << n;
    memset(psi, 0, sizeof(cplx) * dim);
    psi[0] = 1.0;
    orc_noise_t nz = { seed, sigma, 0 };
    int nev = 0;
    for (int l = 0; l < layers; ++l) {
        for (int q = 0; q < n; ++q) {
            double ang[4];
            orc_haar_angles(seed, (uint64_t)l * (uint64_t)n + (uint64_t)q, ang);
            orc_apply_angles(psi, n, &nz, ORC_HAAR, ang, 0, 0, q);
        }
        for (int c = (l & 1); c + 1 < n; c += 2) {
            double ang[2] = { ORC_PI / 2.0, ORC_PI };
            uint64_t cm = (uint64_t)1 << c;
            orc_apply_angles(psi, n, &nz, ORC_RP, ang, cm, cm, c + 1);
        }
        uint64_t all = (n >= 64) ? ~(uint64_t)0 : (((uint64_t)1 << n) - 1);
        orc_inject_paulis(psi, n, seed, (uint64_t)l, all, p, ev, cap, &nev);
    }
    return nev;
}

/* ------------------------------------------------------------------------ */
/* Shor's factoring, semantic mode and classical post-processing             */
/* (PAPER.md:827-859 algorithm box; 896-903 semantic mode; 907-920           */
/* Prob_succ; 969-998 improvements).  SURVEY.md §8(f) row f3.                */
/* ------------------------------------------------------------------------ */

/* ------------------------------------------------------------------------ */
/* Noise experiments, one trajectory each (reading  */
/* R33: trajectory t of a batch with base seed s is exactly the single-      */
/* register circuit below run with seed s + t for both its gate noise and    */
/* its Pauli draws).                                                         */
/* ------------------------------------------------------------------------ */

/* HT experiment (§4.3): start |0..0>; k times: the noisy
 * H = U_R(pi/4 + x) U_P1(pi + y) on every qubit (angle-form RP, gate counter
 * from 0), then the depolarizing channel on every qubit with epoch = the
 * application index (reading R34: one injection point per HT application). */
void orc_traj_ht(cplx *psi, int n, int k, uint64_t seed, double sigma, double p)
{
    const uint64_t dim = (uint64_t)1 << n;
    memset(psi, 0, sizeof(cplx) * dim);
    psi[0] = 1.0;
    orc_noise_t nz = { seed, sigma, 0 };
    const double ang[2] = { ORC_PI / 4.0, ORC_PI };
    for (int i = 0; i < k; ++i) {
        for (int q = 0; q < n; ++q) orc_apply_angles(psi, n, &nz, ORC_RP, ang, 0, 0, q);
        int nev = 0;
        orc_inject_paulis(psi, n, seed, (uint64_t)i, ((uint64_t)1 << n) - 1, p, NULL, 0, &nev);
    }
}

/* Grover experiment (§5.3; reading R35): an n-qubit
 * register (qubits 0..n-1) and the ancilla of V_f (qubit n, the LSB),
 * prepared noiselessly in |0..0>|->.  H_n = noisy RP(pi/4, pi) on every
 * register qubit; V_f = the noisy NOT = RP(pi/2, pi) on the ancilla,
 * controlled by register == f (all n register qubits are controls); one
 * G-iteration = V_{fk}, H_n, V_{f0}, H_n (the global sign -1 is dropped),
 * then the depolarizing channel on every register qubit (epoch = iteration).
 * trace[t] = P(register = k) after iteration t+1 (summed over the ancilla). */
void orc_traj_grover(cplx *psi, int n, uint64_t k, int iters, uint64_t seed, double sigma, double p,
                     double *trace)
{
    const int nt = n + 1;
    const uint64_t dim = (uint64_t)1 << nt;
    memset(psi, 0, sizeof(cplx) * dim);
    const double r = 0.70710678118654752440;
    psi[0] = r;                 /* |0..0>|-> : ancilla (LSB) (|0> - |1>)/sqrt2 */
    psi[1] = -r;
    orc_noise_t nz = { seed, sigma, 0 };
    const double hang[2] = { ORC_PI / 4.0, ORC_PI };
    const double xang[2] = { ORC_PI / 2.0, ORC_PI };
    const uint64_t regmask = ((uint64_t)1 << n) - 1;    /* qubits 0..n-1 */
    for (int q = 0; q < n; ++q) orc_apply_angles(psi, nt, &nz, ORC_RP, hang, 0, 0, q);
    for (int t = 0; t < iters; ++t) {
        /* control values: qubit q (0 = MSB of the register value) has bit n-1-q of f */
        uint64_t vk = 0;
        for (int q = 0; q < n; ++q) vk |= ((k >> (n - 1 - q)) & 1) << q;
        orc_apply_angles(psi, nt, &nz, ORC_RP, xang, regmask, vk, n);
        for (int q = 0; q < n; ++q) orc_apply_angles(psi, nt, &nz, ORC_RP, hang, 0, 0, q);
        orc_apply_angles(psi, nt, &nz, ORC_RP, xang, regmask, 0, n);
        for (int q = 0; q < n; ++q) orc_apply_angles(psi, nt, &nz, ORC_RP, hang, 0, 0, q);
        int nev = 0;
        orc_inject_paulis(psi, nt, seed, (uint64_t)t, regmask, p, NULL, 0, &nev);
        if (trace) {
            const cplx a0 = psi[2 * k], a1 = psi[2 * k + 1];
            trace[t] = creal(a0) * creal(a0) + cimag(a0) * cimag(a0) + creal(a1) * creal(a1) + cimag(a1) * cimag(a1);
        }
    }
}

/* QFT with decoherence (§5.2; reading R36): the QFT
 * circuit of orc_qft on qubits [lo, lo+m) with its angle-form noise, and the
 * depolarizing channel on every qubit of [lo, lo+m) after each R_d gate
 * ("each time the register is applied by the controlled rotation gate R_d"),
 * epoch = the index of that R_d in circuit order (0, 1, ...). */
void orc_qft_decoherent(cplx *psi, int n, int lo, int m, int inverse, orc_noise_t *nz, double p)
{
    const double sgn = inverse ? -1.0 : 1.0;
    const double r = 0.70710678118654752440;
    cplx H[4] = { r, r, r, -r };
    uint64_t qmask = 0;
    for (int q = lo; q < lo + m; ++q) qmask |= (uint64_t)1 << q;
    uint64_t epoch = 0;
    for (int j = 0; j < m; ++j) {
        if (nz->sigma > 0.0) {
            double ang[2] = { ORC_PI / 4.0, ORC_PI };
            orc_apply_angles(psi, n, nz, ORC_RP, ang, 0, 0, lo + j);
        } else {
            orc_apply_1q(psi, n, lo + j, H);
            nz->g += 1;
        }
        for (int k = j + 1; k < m; ++k) {
            double phi = sgn * ORC_PI / ldexp(1.0, k - j);
            uint64_t cm = (uint64_t)1 << (lo + k);
            if (nz->sigma > 0.0) {
                orc_apply_angles(psi, n, nz, ORC_P1, &phi, cm, cm, lo + j);
            } else {
                cplx R[4] = { 1.0, 0.0, 0.0, cos(phi) + I * sin(phi) };
                orc_apply_ctrl(psi, n, cm, cm, lo + j, R);
                nz->g += 1;
            }
            int nev = 0;
            orc_inject_paulis(psi, n, nz->seed, epoch++, qmask, p, NULL, 0, &nev);
        }
    }
    for (int j = 0; j < m / 2; ++j) orc_swap(psi, n, lo + j, lo + m - 1 - j);
}

/* Prob_succ(n) = (1 - phi/(n-1)) + phi/(n-1) * (1/2 * 4/pi^2 * e^-gamma / log log n),
 * natural logarithms. */
double orc_shor_prob_succ(uint64_t n, uint64_t phi)
{
    const double gamma = 0.57721566490153286061;
    const double f = (double)phi / (double)(n - 1);
    return (1.0 - f) + f * (0.5 * 4.0 / (ORC_PI * ORC_PI) * exp(-gamma) / log(log((double)n)));
}

/* Semantic-mode register: the first register is not
 * generated; the second (m qubits, value a) holds the uniform superposition
 * over {a : x^a = v (mod N)}. */
void orc_shor_semantic_state(cplx *psi, int m, uint64_t x, uint64_t N, uint64_t v)
{
    const uint64_t M = (uint64_t)1 << m;
    uint64_t c = 0;
    uint64_t p = 1 % N;
    for (uint64_t a = 0; a < M; ++a) {
        psi[a] = (p == v) ? 1.0 : 0.0;
        c += p == v;
        p = (uint64_t)(((unsigned __int128)p * x) % N);
    }
    const double s = 1.0 / sqrt((double)c);
    for (uint64_t a = 0; a < M; ++a) psi[a] *= s;
}

/* Continued-fraction convergents k/r of y / 2^m (step 4):
 * every convergent with 0 < r < N and |y/2^m - k/r| <= 1/2^(m+1), in order
 * of increasing r.  Returns the count (<= cap). */
int orc_shor_candidates(uint64_t y, int m, uint64_t N, uint64_t *r_out, int cap)
{
    const uint64_t M = (uint64_t)1 << m;
    if (y == 0) return 0;
    /* expansion of y / M with exact integers */
    uint64_t num = y, den = M;
    uint64_t p0 = 0, q0 = 1, p1 = 1, q1 = 0;   /* convergents h_{-2}/k_{-2}, h_{-1}/k_{-1} */
    int cnt = 0;
    while (den != 0) {
        const uint64_t a = num / den;
        const uint64_t t = num - a * den;
        num = den;
        den = t;
        const uint64_t p2 = a * p1 + p0, q2 = a * q1 + q0;
        p0 = p1; q0 = q1; p1 = p2; q1 = q2;
        if (q1 >= N) break;
        if (q1 == 0) continue;
        /* |y/M - p/q| <= 1/(2M)  <=>  |2 (y q - p M)| <= q */
        const __int128 diff = (__int128)y * q1 - (__int128)p1 * M;
        const __int128 ad = diff < 0 ? -diff : diff;
        if (2 * ad <= (__int128)q1 && p1 > 0 && cnt < cap) r_out[cnt++] = q1;
    }
    return cnt;
}

/* Steps 4-5 for one candidate r.  gcd_check = 1 is the
 * "GCD Check" improvement: d+- are tried even when
 * x^r != 1.  Returns a nontrivial factor of N or 0. */
uint64_t orc_shor_try(uint64_t N, uint64_t x, uint64_t r, int gcd_check)
{
    if (r == 0 || (r & 1)) return 0;
    const uint64_t xr = orc_powmod(x, r, N);
    if (xr != 1 % N && !gcd_check) return 0;
    const uint64_t z = orc_powmod(x, r / 2, N);
    if (!gcd_check && (z == 1 % N || z == N - 1)) return 0;
    const uint64_t d1 = orc_gcd(N, (z + N - 1) % N), d2 = orc_gcd(N, (z + 1) % N);
    if (d1 > 1 && d1 < N) return d1;
    if (d2 > 1 && d2 < N) return d2;
    return 0;
}

static uint64_t lcm64(uint64_t a, uint64_t b) { return a / orc_gcd(a, b) * b; }

/* Tallies of one or more runs (Table 6: "s/f where s
 * means the number of success iterations and f ... failure iterations"). */
enum { ST_STEP2 = 0, ST_QUANTUM, ST_BASIC_S, ST_BASIC_F, ST_NEIGH_S, ST_NEIGH_F, ST_GCD_S, ST_GCD_F,
       ST_SF_S, ST_SF_F, ST_LCM_S, ST_LCM_F, ST_COUNT };

/* The post-processing of one measured y (R27):
 *   candidate r from the continued fraction of y/2^m (step 4); none and
 *   improved: Neighbor y Check -- y+1, y-1, y+2, y-2, first with a candidate
 *   (success = a candidate found);
 *   basic test of step 5 on r;
 *   improved, r even: GCD Check -- d+- even if x^r != 1;
 *   improved, x^r != 1: Small Factor Check -- k r for k = 2..8 with the
 *   basic test and the GCD check;
 *   improved, earlier candidates r1: LCM Check -- lcm(r1, r) likewise;
 *   r is remembered for later LCM checks. */
static uint64_t shor_post(uint64_t N, int m, uint64_t x, uint64_t y, int improved,
                          uint64_t *mem, int *nmem, int64_t *st)
{
    const uint64_t M = (uint64_t)1 << m;
    uint64_t rs[64];
    int nr = y ? orc_shor_candidates(y, m, N, rs, 64) : 0;
    if (nr == 0) {
        if (!improved) return 0;
        const int64_t dy[4] = { 1, -1, 2, -2 };
        for (int i = 0; i < 4 && nr == 0; ++i) {
            const int64_t yy = (int64_t)y + dy[i];
            if (yy > 0 && (uint64_t)yy < M) nr = orc_shor_candidates((uint64_t)yy, m, N, rs, 64);
        }
        st[nr ? ST_NEIGH_S : ST_NEIGH_F]++;
        if (nr == 0) return 0;
    }
    const uint64_t r = rs[nr - 1];
    uint64_t f = orc_shor_try(N, x, r, 0);
    st[f ? ST_BASIC_S : ST_BASIC_F]++;
    if (f || !improved) return f;
    if (r % 2 == 0) {
        f = orc_shor_try(N, x, r, 1);
        st[f ? ST_GCD_S : ST_GCD_F]++;
        if (f) return f;
    }
    if (orc_powmod(x, r, N) != 1 % N) {
        for (uint64_t k = 2; k <= 8 && !f; ++k) {
            f = orc_shor_try(N, x, k * r, 0);
            if (!f) f = orc_shor_try(N, x, k * r, 1);
        }
        st[f ? ST_SF_S : ST_SF_F]++;
        if (f) return f;
    }
    if (*nmem > 0) {
        for (int j = 0; j < *nmem && !f; ++j) {
            const uint64_t l = lcm64(mem[j], r);
            f = orc_shor_try(N, x, l, 0);
            if (!f) f = orc_shor_try(N, x, l, 1);
        }
        st[f ? ST_LCM_S : ST_LCM_F]++;
        if (f) return f;
    }
    if (*nmem < 64) mem[(*nmem)++] = r;
    return 0;
}

/* One factoring run (PAPER.md:827-859 repeated until a factor is found,
 * PAPER.md:928-930): iteration t draws (a, b) = draw(seed, TAG_SHOR, run,
 * t-1): x = 1 + uint(a, N-1) (step 1); step 2: 1 < gcd(x, N) < N ends the
 * run; else the semantic order-finding register for the
 * first-register outcome v = x^uint(b, 2^m) mod N, the QFT,
 * measurement y with r = u01(draw(seed, TAG_MEASURE, run, t-1).a)
 * (PAPER.md:397-404), then shor_post.  Returns the iteration count (0: none
 * within max_iter); *factor receives the factor; st (ST_COUNT int64, may be
 * NULL) accumulates the tallies. */
int orc_shor_run(uint64_t N, int m, uint64_t seed, uint64_t run, int improved, int max_iter, uint64_t *factor,
                 int64_t *stats)
{
    const uint64_t M = (uint64_t)1 << m;
    cplx *psi = (cplx *)malloc(sizeof(cplx) * M);
    uint64_t mem[64];
    int nmem = 0;
    int64_t local[ST_COUNT] = { 0 };
    int64_t *st = stats ? stats : local;
    *factor = 0;
    for (int t = 1; t <= max_iter; ++t) {
        uint64_t d[2];
        orc_draw(seed, TAG_SHOR, run, (uint32_t)(t - 1), d);
        const uint64_t x = 1 + orc_uint(d[0], N - 1);
        const uint64_t g = orc_gcd(x, N);
        if (g > 1 && g < N) { st[ST_STEP2]++; *factor = g; free(psi); return t; }
        st[ST_QUANTUM]++;
        const uint64_t v = orc_powmod(x, orc_uint(d[1], M), N);
        orc_shor_semantic_state(psi, m, x, N, v);
        orc_noise_t nz = { 0, 0.0, 0 };
        orc_qft(psi, m, 0, m, 0, &nz);
        uint64_t dm[2];
        orc_draw(seed, TAG_MEASURE, run, (uint32_t)(t - 1), dm);
        const uint64_t y = orc_measure(psi, m, orc_u01(dm[0]));
        const uint64_t f = shor_post(N, m, x, y, improved, mem, &nmem, st);
        if (f) { *factor = f; free(psi); return t; }
    }
    free(psi);
    return 0;
}

/* Host threads the oracle's parallel loops use (results are bit-identical for
 * any count); 0 restores the OpenMP default.  Timing only (bench.py). */
void orc_set_threads(int k)
{
    omp_set_num_threads(k > 0 ? k : omp_get_num_procs());
}

int orc_get_threads(void) { return omp_get_max_threads(); }
