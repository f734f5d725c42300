/*
 * qsim.h -- C-ABI of libqsim.so, the B200-native (sm_100a) state-vector gate
 * engine for the method of Niwa, Matsumoto, Imai, "General-Purpose Parallel
 * Simulator for Quantum Computing" (arXiv quant-ph/0201042; PAPER.md).
 *
 * Conventions (all entry points):
 *   - Status: QSIM_OK (0) or a negative QSIM_E* code; qsim_last_error() has
 *     the message.  Validation happens before anything is enqueued, so a
 *     failed call has no effect on the state.  A CUDA or NCCL failure poisons
 *     the handle: every later call returns QSIM_ESTATE.
 *   - Qubits (§2.2.1): qubit 0 is the MSB; qubit q of an n-qubit
 *     register is bit (n-1-q) of the basis index.  Qubit sets (ctrl_mask,
 *     ctrl_vals, qubit masks) are bit sets over qubit numbers: bit q <-> qubit q.
 *   - Amplitudes are complex128, qsim_c128 = {re, im}, layout-compatible with
 *     double2 / std::complex<double> / numpy complex128 (2^(n+4)
 *     bytes per state; reading R2 in DESIGN.md).
 *   - Host pointers are borrowed for the duration of the call only; the
 *     caller owns every buffer it passes.  The handle owns all device memory,
 *     streams and communicators.
 *   - Gate calls are asynchronous and stream-ordered on the handle's stream;
 *     calls that return data to the host (norm, probs, get_state, measure,
 *     sync, inject_errors' event list) synchronise that stream.
 *   - A handle is not thread-safe: one mutator at a time.
 *   - Multi-GPU: qsim_create(n, ngpus) / qsim_create_group (one process
 *     drives every GPU) or one process per GPU (qsim_create_dist).  The state is sharded
 *     on its top log2(world) physical bits; the library tracks a logical ->
 *     physical qubit map internally, exchanges shards with NCCL send/recv when
 *     a gate needs a global qubit local, and restores the canonical layout
 *     before any call that exposes amplitudes or marginals.  Every rank must
 *     make the same sequence of calls (SPMD).
 * The semantics of each call are pinned by the CPU oracle (oracle/, test
 * infrastructure) as described in DESIGN.md §4.
 */
#ifndef QSIM_H
#define QSIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qsim_s qsim_t;

typedef struct { double re, im; } qsim_c128;

enum {
    QSIM_OK = 0,
    QSIM_EINVAL = -1,     /* malformed argument (overlapping qubits, p outside [0,1], ...) */
    QSIM_ERANGE = -2,     /* qubit / index / size outside the register */
    QSIM_ENOMEM = -3,     /* device or pinned allocation failed */
    QSIM_ECUDA = -4,      /* CUDA runtime error (handle poisoned) */
    QSIM_ENOTBIJ = -5,    /* permutation is not a bijection */
    QSIM_ESTATE = -6,     /* handle poisoned by an earlier asynchronous error */
    QSIM_ENCCL = -7,      /* NCCL error (handle poisoned) */
    QSIM_ENODEV = -8,     /* no CUDA device / not an sm_100 device */
    QSIM_ENONUNITARY = -9 /* strict mode (qsim_set_strict): the matrix is not unitary */
};

/* Angle-form gate kinds (§3.2; R12-R14).
 *   QSIM_GATE_RP   : U_R(a0) U_P1(a1)                 (H = RP(pi/4, pi), NOT = RP(pi/2, pi))
 *   QSIM_GATE_P1   : U_P1(a0) = diag(1, e^{i a0})      (R_d = P1(pi / 2^d))
 *   QSIM_GATE_HAAR : U_P2(a0) U_P1(a1) U_R(a2) U_P1(a3) (general single-qubit gate)
 * with U_R(t) = (cos t, -sin t; sin t, cos t), U_P1(p) = diag(1, e^{ip}),
 * U_P2(p) = diag(e^{ip}, 1). */
enum { QSIM_GATE_RP = 0, QSIM_GATE_P1 = 1, QSIM_GATE_HAAR = 2 };

/* Counter-RNG tags (R1). */
enum {
    QSIM_TAG_GATE = 1, QSIM_TAG_HAAR = 2, QSIM_TAG_PAIR = 3, QSIM_TAG_OPNOISE = 4,
    QSIM_TAG_MARK = 5, QSIM_TAG_BASE = 6, QSIM_TAG_GAUSS = 7, QSIM_TAG_PAULI = 8,
    QSIM_TAG_MEASURE = 9, QSIM_TAG_SHOR = 10
};

/* ---------------------------------------------------------------- lifecycle */

/* Allocate an n-qubit register (2^(n+4) bytes of HBM),
 * initialised to |0...0>.  ngpus = 1: on the current CUDA device.  ngpus > 1
 * (a power of two): sharded over CUDA devices 0..ngpus-1 on its top
 * log2(ngpus) qubits, all driven by this process -- the same handle as
 * qsim_create_group(n, ngpus, {0, 1, ..., ngpus-1}); when fewer devices are
 * visible, rank r goes to device r mod (device count).  The paper's pairing
 * of rows R_j / R_{2^P + j} across processors (§2.2.1) is
 * what the shard exchanges implement.  Errors: QSIM_ERANGE if n < 1, n > 40
 * or 2^n < 2 ngpus; QSIM_EINVAL if ngpus is not a power of two in [1, 64];
 * QSIM_ENOMEM (message names the byte count); QSIM_ENODEV.  *out receives
 * the handle (NULL on error; qsim_last_error(NULL) then has the message). */
int qsim_create(int n, int ngpus, qsim_t **out);

/* One rank of a world of `world` processes (world a power of two, one GPU
 * each, 2^n >= 2*world): allocates this rank's shard of 2^(n - log2 world)
 * amplitudes on CUDA device `device` and joins the NCCL communicator named by
 * the 128-byte `nccl_id` (from qsim_nccl_unique_id on rank 0, broadcast by
 * the caller).  State = |0...0>.  Errors as qsim_create, plus QSIM_ENCCL. */
int qsim_create_dist(int n, int world, int rank, int device, const void *nccl_id,
                     qsim_t **out);

/* All `world` ranks in this process (world a power of two): one shard per
 * rank on devices[r] (devices may be NULL: the current device for every
 * rank; ranks may share a device).  The returned group handle accepts every
 * call; each call runs on all ranks, shard exchanges are device-to-device
 * copies (peer copies over NVLink between GPUs) instead of NCCL, and
 * qsim_get_state / qsim_set_state address every slice.  Same layout and
 * exchange plan as qsim_create_dist. */
int qsim_create_group(int n, int world, const int *devices, qsim_t **out);

/* Writes a fresh ncclUniqueId (128 bytes) into out128. */
int qsim_nccl_unique_id(void *out128);

/* Frees every device buffer, stream and communicator of the handle. */
void qsim_destroy(qsim_t *h);

/* Message of the last failed call on h (h may be NULL for creation errors). */
const char *qsim_last_error(const qsim_t *h);

/* 2^(n+4): bytes of an n-qubit complex128 state. */
uint64_t qsim_memory_bytes(int n);

/* Number of this library's kernels launched on h so far (instrumentation). */
uint64_t qsim_launch_count(const qsim_t *h);

/* Waits for all queued work on h and surfaces asynchronous errors. */
int qsim_sync(qsim_t *h);

/* The cudaStream_t (as void*) every kernel of h is launched on, so callers
 * can record CUDA events on it (plumbing for timing; do not destroy it). */
void *qsim_get_stream(qsim_t *h);

/* Strict mode (default off): qsim_apply_1q / qsim_apply_ctrl (and matrix
 * entries of qsim_apply_gates) return QSIM_ENONUNITARY, with no effect, when
 * max |(U U^dagger - I)_rc| > 1e-12 -- the paper's gates are unitary
 * (§2.2.1).  Off, any 2x2 matrix is applied as given. */
int qsim_set_strict(qsim_t *h, int enable);

/* Gate fusion (default on for shards of >= 2^9 amplitudes): single-qubit
 * and controlled gates are queued and applied as fused tile passes (one HBM
 * read + write for a run of gates) when anything else is called or at
 * qsim_sync.  enable = 0 runs every gate as its own kernel (flushes first). */
int qsim_set_fusion(qsim_t *h, int enable);

/* Per-launch profiling: with enable = 1 every kernel launch of h is
 * bracketed by CUDA events on h's stream (records are reset by each call).
 * qsim_profile_json synchronises and returns, aggregated per kernel name,
 * {"name": {"launches": L, "ms": total device time, "bytes": algorithmic
 * HBM bytes (reads + writes the operation must make)}, ...}; the string is
 * owned by h and valid until the next call. */
int qsim_profile(qsim_t *h, int enable);
const char *qsim_profile_json(qsim_t *h);

/* ---------------------------------------------------------------- state preparation */

/* |idx> (registers start in basis states).  QSIM_ERANGE if
 * idx >= 2^n. */
int qsim_set_basis(qsim_t *h, uint64_t idx);

/* i.i.d. complex Gaussian amplitudes, then divided by sqrt(sum |a|^2)
 * (BASELINE configs[2]; R19): amplitude idx is the Box-Muller pair
 * of draw(seed, GAUSS, idx, 0), re = cos branch, im = sin branch.  Generated
 * on the device by the library's own Philox4x32-10. */
int qsim_init_gaussian(qsim_t *h, uint64_t seed);

/* Copy cnt amplitudes starting at global basis index off between the state
 * and a caller-owned host buffer (canonical order).  Synchronising.
 * QSIM_ERANGE if off + cnt > 2^n.  In a distributed handle only the indices
 * owned by this rank ([rank * 2^nl, (rank+1) * 2^nl)) may be addressed. */
int qsim_set_state(qsim_t *h, uint64_t off, uint64_t cnt, const qsim_c128 *host);
int qsim_get_state(qsim_t *h, uint64_t off, uint64_t cnt, qsim_c128 *host);

/* ---------------------------------------------------------------- gates (§2.2) */

/* Single-qubit gate U (row-major u11, u12, u21, u22, copied at call time) on
 * qubit q: the pair (j, j + 2^(n-1-q)) with bit (n-1-q)
 * of j clear becomes (u11 a + u12 b, u21 a + u22 b), in place
 * (PAPER.md:285-337).  Unitarity is not checked.  QSIM_ERANGE if q not in
 * [0, n). */
int qsim_apply_1q(qsim_t *h, int q, const qsim_c128 U[4]);

/* Controlled gate: the pair update of qsim_apply_1q only
 * where every qubit c in ctrl_mask has value bit c of ctrl_vals ("the c-th
 * bit in j is 1" generalised to several controls and either value; all-ones
 * ctrl_vals is the standard controlled-U; CNOT is U = NOT).  QSIM_EINVAL if q
 * is in ctrl_mask or ctrl_vals has bits outside ctrl_mask. */
int qsim_apply_ctrl(qsim_t *h, uint64_t ctrl_mask, uint64_t ctrl_vals, int q,
                    const qsim_c128 U[4]);

/* Angle-form gate (kinds above), optionally controlled (ctrl_mask = 0 for
 * none).  With gate noise enabled (qsim_set_gate_noise, sigma > 0) angle slot
 * s is perturbed by sigma * z, z = normal(draw(noise_seed, OPNOISE, g, s))
 * (R15), g = the handle's angle-form gate
 * counter, which advances by one per call whatever sigma is.  ang holds 2, 1
 * or 4 angles for RP, P1, HAAR. */
int qsim_apply_angles(qsim_t *h, int kind, const double *ang, uint64_t ctrl_mask,
                      uint64_t ctrl_vals, int q);

/* Operational-error model (§3.2): sigma >= 0 (QSIM_EINVAL
 * otherwise); sigma = 0 disables.  Does not reset the gate counter. */
int qsim_set_gate_noise(qsim_t *h, uint64_t seed, double sigma);
int qsim_get_gate_counter(const qsim_t *h, uint64_t *g);
int qsim_set_gate_counter(qsim_t *h, uint64_t g);

/* SWAP of qubits q1, q2 (the closing swaps of the QFT circuit, R7).
 * Exact (a permutation of amplitudes). */
int qsim_swap(qsim_t *h, int q1, int q2);

/* Hadamard transform H on every qubit of [lo, lo+m) (PAPER.md:420-436,
 * §2.3.1), with the constant H = (1/sqrt2)(1 1; 1 -1). */
int qsim_hadamard(qsim_t *h, int lo, int m);

/* H on every qubit of [lo, lo+m) as the paper's angle-form gate
 * H = U_R(pi/4) U_P1(pi) (the H of its noisy circuits,
 * PAPER.md:738-747): exactly the m calls qsim_apply_angles(h,
 * QSIM_GATE_RP, {pi/4, pi}, 0, 0, q) for q = lo .. lo+m-1 -- with gate noise
 * each H draws its two angle perturbations from the gate counter, which
 * advances by m.  Executed as fused HBM passes where the register allows
 * (single GPU, no trajectory batch), else gate by gate.  QSIM_ERANGE if the
 * range leaves [0, n). */
int qsim_hadamard_angles(qsim_t *h, int lo, int m);

/* QFT (inverse = 0) or inverse QFT (inverse = 1) on the sub-register of
 * qubits [lo, lo+m), qubit lo its MSB (§2.3.2; DESIGN.md
 * R6-R8): beta_x = 2^(-m/2) sum_y e^(+-2 pi i x y / 2^m) alpha_y on the
 * sub-register value, computed as the circuit H(lo+j), R_{k-j} controlled by
 * lo+k on lo+j (k > j), closing swaps.  Without gate noise the gates are the
 * constant matrices and the whole circuit runs as fused HBM passes; with gate
 * noise every H / R_d is an angle-form gate (counter advances per H and R_d,
 * m + m(m-1)/2 in total either way) -- still fused passes carrying each
 * gate's perturbed matrix / angle on a single GPU (R38), gate by
 * gate otherwise.  QSIM_ERANGE if the range leaves [0, n). */
int qsim_qft(qsim_t *h, int lo, int m, int inverse);

/* FFT of the sub-register [lo, lo+m) ("If we regard the
 * QFT transform as a black box operator ... we can use fast Fourier
 * transform (FFT) in the simulator instead of the QFT circuit"; SURVEY §8(f)
 * row f1): the exact transform beta_x = 2^(-m/2) sum_y e^(+-2 pi i x y/2^m)
 * alpha_y of qsim_qft, never subject to gate noise and not counted by the
 * gate counter (it is not a circuit).  Radix-2^(<=10) Cooley-Tukey passes over
 * HBM (the same tile kernels as the noiseless QFT).  QSIM_ERANGE if the range
 * leaves [0, n). */
int qsim_fft(qsim_t *h, int lo, int m, int inverse);

/* Approximate QFT (§2.3.2; Barenco et al.; R30):
 * the qsim_qft circuit with every R_d of distance d = k - j > b left out.
 * b >= m-1 is qsim_qft.  Gate noise applies as in qsim_qft; the gate counter
 * advances only for the gates that are applied.  Executed as fused HBM
 * passes with the gates' own matrices and angles (single GPU, no trajectory
 * batch, >= 4 and <= local-qubit wires), else gate by gate.  QSIM_ERANGE if
 * the range leaves [0, n) or b < 0. */
int qsim_aqft(qsim_t *h, int lo, int m, int b, int inverse);

/* The QFT (as qsim_qft, noiseless) of `count` host-resident states, end to
 * end and pipelined: state i is in[i * in_stride .. + 2^n) and its transform
 * goes to out[i * out_stride .. + 2^n) (strides in amplitudes; 0 reuses one
 * buffer).  State i+1 is copied to the device on one stream while state i is
 * transformed and state i-1 copied back on another, through four device shard
 * buffers (the state, the scratch and two stages: 4 x 2^(n+4) bytes).  Use
 * pinned host memory for the copies to overlap.  The handle's state becomes
 * the last result.  Synchronising.  Single-GPU handles without gate noise;
 * QSIM_EINVAL otherwise, QSIM_ERANGE on the range, QSIM_ENOMEM. */
int qsim_qft_host_stream(qsim_t *h, int lo, int m, int inverse, const qsim_c128 *in, uint64_t in_stride,
                         qsim_c128 *out, uint64_t out_stride, int count);

/* Sign-changing operator V_f for f = delta_{x, idx}, as
 * the phase flip alpha_idx <- -alpha_idx (R17).  QSIM_ERANGE if
 * idx >= 2^n. */
int qsim_phase_flip(qsim_t *h, uint64_t idx);

/* Diffusion D = -H_m V_{f0} H_m = 2|s><s| - I on the sub-register [lo, lo+m)
 * (§5.3; |s> = H_m|0>, the sign kept literally): for
 * every value of the other qubits, alpha_y <- 2 mean_y(alpha) - alpha_y.  The
 * whole register (lo = 0, m = n) runs in the mean form (one read pass for the
 * fixed-order sum, one update pass; shards summed on the host in rank order);
 * a sub-register runs the literal H_m, diagonal 2|0><0| - I, H_m as fused
 * passes.  Asynchronous except for the whole-register sum.  QSIM_ERANGE if
 * the range leaves [0, n) or m < 1. */
int qsim_diffusion(qsim_t *h, int lo, int m);

/* Grover's search on the whole register (§5.3): `iters`
 * G-iterations -H_n V_{f0} H_n V_{fk} with f_k = delta_{x, mark}, applied in
 * the equivalent form alpha_k <- -alpha_k; alpha <- 2 mean(alpha) - alpha.
 * trace (host, iters doubles, may be NULL) receives |alpha_mark|^2 after each
 * iteration.  One GPU: all iterations in one cooperative kernel.  Sharded
 * handles: qsim_phase_flip + qsim_diffusion(0, n) per iteration.
 * Synchronising when trace != NULL. */
int qsim_grover(qsim_t *h, uint64_t mark, int iters, double *trace);

/* ---------------------------------------------------------------- permutations (§2.3.3) */

enum { QSIM_PERM_TABLE = 0, QSIM_PERM_MODMUL = 1, QSIM_PERM_MODEXP = 2 };

/* A basis permutation, given as data:
 *   TABLE : target register [lo, lo+m) (m <= 24), table[v] = image of value v
 *           (2^m entries, must be a bijection), applied where the control
 *           qubits match (ctrl_mask / ctrl_vals as in qsim_apply_ctrl).
 *   MODMUL: target register [lo, lo+m): v -> v*mult mod modulus for v < modulus,
 *           identity for v >= modulus (R10); gcd(mult, modulus) = 1,
 *           modulus <= 2^m; controlled as above.
 *   MODEXP: work register [lo, lo+m), exponent register [elo, elo+em) (value e,
 *           qubit elo its MSB): v -> v * base^e mod modulus (v < modulus) --
 *           the whole chain of controlled multiplications by base^(2^i)
 *            applied at once.  gcd(base, modulus) = 1.
 * Registers must not overlap (QSIM_EINVAL); a non-bijective table or
 * gcd != 1 gives QSIM_ENOTBIJ. */
typedef struct {
    int kind;
    int lo, m;
    int elo, em;
    uint64_t ctrl_mask, ctrl_vals;
    uint64_t mult, base, modulus;
    const uint32_t *table;
} qsim_perm_t;

int qsim_apply_perm(qsim_t *h, const qsim_perm_t *f);

/* ---------------------------------------------------------------- decoherence (§3.1) */

typedef struct {
    double p;             /* depolarizing probability per qubit, in [0, 1] */
    uint64_t qubit_mask;  /* qubits that see the channel */
    uint64_t epoch;       /* injection point (counter i of the draws) */
} qsim_noise_t;

typedef struct {
    uint64_t epoch;
    int32_t qubit;
    int32_t pauli;   /* 1 X, 2 Y, 3 Z */
    uint64_t traj;   /* trajectory of a batched handle (qsim_set_batch), else 0 */
} qsim_event_t;

/* Depolarizing channel on pure-state trajectories: for each
 * qubit q in qubit_mask (ascending), u = u01(draw(seed, PAULI, epoch, q).a);
 * u < p/3 -> sigma_x, u < 2p/3 -> sigma_y, u < p -> sigma_z (R16),
 * applied to the state.  Events are written to ev (capacity cap, may be NULL)
 * in qubit order and *nev (may be NULL) receives the event count.
 * QSIM_EINVAL if p not in [0, 1]; QSIM_ERANGE if the events did not fit (they
 * are still applied). */
int qsim_inject_errors(qsim_t *h, uint64_t seed, const qsim_noise_t *model,
                       qsim_event_t *ev, int cap, int *nev);

/* ---------------------------------------------------------------- read-out */

/* sum_i |alpha_i|^2, tree-summed on the device. */
int qsim_norm(qsim_t *h, double *out);

/* Marginal probabilities of the sub-register [lo, lo+m) (qubit lo = MSB of
 * the value y): out[y] = sum of |alpha_j|^2 over j with sub-register value y.
 * out is a caller-owned host buffer of 2^m doubles (m <= 26). */
int qsim_probs(qsim_t *h, int lo, int m, double *out);

/* |alpha_idx|^2 of one amplitude. */
int qsim_prob_index(qsim_t *h, uint64_t idx, double *out);

/* Measurement (§2.2.3) without collapse: for r in [0, 1),
 * the smallest i with sum_{j<=i} |alpha_j|^2 > r (block sums on the device,
 * then a scan of one block); if rounding leaves r >= the total, the largest i
 * with alpha_i != 0 (R22). */
int qsim_measure(qsim_t *h, double r, uint64_t *idx);

/* Measurement of the sub-register [lo, lo+m) (PAPER.md:391-404 applied to
 * its marginal distribution; R31): y = the smallest value with
 * sum_{y'<=y} P(y') > r (P as qsim_probs, summed in order on the host); if
 * rounding leaves r >= the total, the largest y with P(y) > 0.  With
 * collapse != 0 the state is projected onto y and renormalised by
 * 1/sqrt(P(y)) on the device.  m <= 26.  Synchronising. */
int qsim_measure_range(qsim_t *h, int lo, int m, double r, int collapse, uint64_t *y);

/* Inner product <a|b> = sum_i conj(a_i) b_i of two registers of the same size
 * on the same devices (the paper's fidelity is its modulus, "the inner product
 * of the correct state and the simulated state"; DESIGN.md
 * R32).  Fixed-order tree sums on the device, ranks combined in rank order.
 * QSIM_EINVAL if the handles differ in n, world or devices.  Synchronising. */
int qsim_inner(qsim_t *a, qsim_t *b, qsim_c128 *out);

/* ---------------------------------------------------------------- batched trajectories */
/* Batched noisy trajectories (R33): the
 * top b qubits [0, b) of the handle index 2^b independent trajectories of
 * the register [b, n) -- the paper's noise experiments average 1000-10000
 * runs.  Trajectory t draws its gate
 * noise (qsim_set_gate_noise seed s) from s + t and its Pauli events
 * (qsim_inject_errors seed s) from s + t, so it is exactly the single-register
 * circuit run with seed s + t.  Gates may not act on [0, b); angle-form gates
 * with sigma > 0 get one matrix per trajectory (built on the device), Pauli
 * injection gives one event list over all trajectories (qubit order, then
 * trajectory order, event.traj = t).  qsim_probs over [b, n) is the average
 * over trajectories of each trajectory's marginal.  b must cover the rank
 * bits of a sharded handle (trajectories shard across GPUs with no data
 * exchange); n - b >= 9; b <= 24.  b = 0 turns batching off.  Flushes. */
int qsim_set_batch(qsim_t *h, int b);

/* Every trajectory set to the register state reg (host, 2^(n-b) amplitudes,
 * normalised by the caller); amplitudes are stored scaled by 2^(-b/2) so the
 * whole handle has norm 1.  Resets the layout.  QSIM_EINVAL if not batched. */
int qsim_batch_set_state(qsim_t *h, const qsim_c128 *reg);

/* out[t] = <ref|psi_t> for every trajectory t (host buffers: ref 2^(n-b)
 * amplitudes, out 2^b values); the paper's fidelity is |out[t]| averaged
 * (R32).  Fixed-order tree per trajectory.  Synchronising. */
int qsim_batch_overlap(qsim_t *h, const qsim_c128 *ref, qsim_c128 *out);

/* ---------------------------------------------------------------- Shor, semantic mode */
/* Shor's factoring algorithm in the paper's semantic mode
 * (modular exponentiation classical, first register not
 * generated, QFT by the fast transform).  The exponent register is the whole
 * handle: m = n = 2l qubits for an l-bit modulus, value a = basis index. */

/* Prepare the post-measurement exponent register of step 3: the uniform
 * superposition over {a < 2^n : x^a = v (mod N)}, amplitude 1/sqrt(count)
 * (the predicate and the count are evaluated on the device).  Resets the
 * layout to canonical and discards queued gates.  QSIM_ERANGE unless
 * 3 <= N < 2^32; QSIM_EINVAL if x >= N or v >= N, or if no exponent matches
 * (state then undefined). */
int qsim_shor_semantic_state(qsim_t *h, uint64_t x, uint64_t N, uint64_t v);

/* Tallies of qsim_shor_run (Table 6: s/f = iterations in
 * which a check was performed and succeeded / failed). */
enum {
    QSIM_SHOR_STEP2 = 0,      /* runs ended by step 2 (1 < gcd(x, N) < N) */
    QSIM_SHOR_QUANTUM = 1,    /* iterations that ran the order-finding register */
    QSIM_SHOR_BASIC_S = 2, QSIM_SHOR_BASIC_F = 3,        /* step 5 on the candidate */
    QSIM_SHOR_NEIGHBOR_S = 4, QSIM_SHOR_NEIGHBOR_F = 5,  /* 1 (Neighbor): a candidate found */
    QSIM_SHOR_GCD_S = 6, QSIM_SHOR_GCD_F = 7,            /* 2 (GCD): a factor found */
    QSIM_SHOR_SF_S = 8, QSIM_SHOR_SF_F = 9,              /* 3 (Small Factor) */
    QSIM_SHOR_LCM_S = 10, QSIM_SHOR_LCM_F = 11,          /* 4 (LCM) */
    QSIM_SHOR_NSTATS = 12
};

/* One factoring run: repeat the algorithm until a nontrivial factor of N is
 * found or max_iter iterations have run.  Iteration t
 * (1-based) draws (a, b) = draw(seed, QSIM_TAG_SHOR, run, t-1):
 * x = 1 + uint(a, N-1); if 1 < gcd(x, N) < N step 2 succeeds; otherwise
 * v = x^(uint(b, 2^n)) mod N (the outcome of measuring f(a) = x^a mod N),
 * qsim_shor_semantic_state, qsim_qft(0, n), and y = qsim_measure(u01(
 * draw(seed, QSIM_TAG_MEASURE, run, t-1).a)); then steps 4-5 on y.
 * improved = 1 adds the four checks of PAPER.md:969-998 in the paper's order
 * (R27).  *iters = t of the success, 0 if none (then *factor = 0).
 * stats: NULL or a host array of QSIM_SHOR_NSTATS counters, incremented
 * (not reset).  Overwrites the state.  QSIM_ERANGE unless 3 <= N < 2^32 and
 * N^2 <= 2^n (the precision of PAPER.md:841-843). */
int qsim_shor_run(qsim_t *h, uint64_t N, uint64_t seed, uint64_t run, int improved, int max_iter,
                  uint64_t *factor, int *iters, int64_t *stats);

/* Step 4's classical part: every convergent k/r of the
 * continued fraction of y / 2^m with 0 < k, 0 < r < N and
 * |y/2^m - k/r| <= 1/2^(m+1), in order of increasing r.  Writes up to cap
 * denominators to r_out (host); returns their number, or QSIM_EINVAL. */
int qsim_shor_candidates(uint64_t y, int m, uint64_t N, uint64_t *r_out, int cap);

/* Step 5 for one candidate r: 0 (failure) if r is odd,
 * x^r != 1 or x^(r/2) = -1 (mod N) ... else the nontrivial one of
 * d+- = gcd(N, x^(r/2) +- 1).  gcd_check = 1 is the "GCD Check" of
 * d+- are tried for every even r. */
uint64_t qsim_shor_try(uint64_t N, uint64_t x, uint64_t r, int gcd_check);

/* Prob_succ(N) of PAPER.md:907-920 for phi = phi(N), natural logarithms;
 * 1 / Prob_succ is Table 5's "Theoretical" column.
 * NaN unless 3 <= N and 0 < phi < N. */
double qsim_shor_prob_succ(uint64_t N, uint64_t phi);

/* ---------------------------------------------------------------- counter RNG */

/* The library's own Philox4x32-10 draw (R1), exported so that
 * callers can generate circuits from the same seeds: key = (seed lo, seed hi),
 * counter = (i lo, i hi, j, tag); out[0] = x0 | x1 << 32, out[1] = x2 | x3 << 32. */
void qsim_philox_draw(uint64_t seed, uint32_t tag, uint64_t i, uint32_t j, uint64_t out[2]);

/* count consecutive draws: out[2k], out[2k+1] = qsim_philox_draw(seed, tag,
 * i0 + k, j) for k < count (caller-owned buffer of 2 * count words). */
void qsim_philox_draws(uint64_t seed, uint32_t tag, uint64_t i0, uint64_t count, uint32_t j, uint64_t *out);

/* ---------------------------------------------------------------- gate lists */

/* One queued gate: type QSIM_GT_MATRIX applies U to qubit q (controlled by
 * ctrl_mask / ctrl_vals when ctrl_mask != 0) exactly as qsim_apply_1q /
 * qsim_apply_ctrl; type QSIM_GT_ANGLES applies the angle-form gate `akind`
 * (QSIM_GATE_*) with angles ang[] as qsim_apply_angles (gate noise and the
 * gate counter included). */
enum { QSIM_GT_MATRIX = 0, QSIM_GT_ANGLES = 1 };
typedef struct {
    int type;
    int q;
    int akind;
    int pad_;
    uint64_t ctrl_mask, ctrl_vals;
    double ang[4];
    qsim_c128 U[4];
} qsim_gate_t;

/* Apply gates[0 .. count) in order, as the corresponding single calls would
 * (one C-ABI crossing for a whole circuit).  Stops at the first invalid gate:
 * its error code is returned, *done (if not NULL) = the number applied before
 * it. */
int qsim_apply_gates(qsim_t *h, const qsim_gate_t *gates, int count, int *done);

/* ---------------------------------------------------------------- host-only exchange planner */

/* The planner behind every shard exchange (no device work; exposed for the
 * multi-process CPU tests).  The paper's large-subblock rule (PAPER.md:264-289,
 * §2.2.1: rows R_j and R_{2^P + j} must meet on one processor) becomes a list
 * of steps on the physical layout of an n-qubit state over `world` ranks
 * (world a power of two), written as int triples (kind, a, b) into
 * steps[0 .. 3*cap):
 *   kind 0 LSWAP (a, b): swap local positions a and b;
 *   kind 1 XCHG  (g, -): swap rank-bit position g with the top local position
 *                        (rank r trades half its shard with rank r ^ 2^(g - nl));
 *   kind 2 A2A   (k, -): swap the k rank-bit positions with the top k local
 *                        positions in one all-to-all.
 * pos_io (n ints: logical qubit -> physical position, caller-owned) is
 * updated as the steps move the data.  qsim_plan_make_local plans for the
 * nneed logical qubits in need (caller-owned) to become local;
 * qsim_plan_canonical_globals for the rank bits to hold qubits 0..log2(world)-1
 * again.  Return the number of steps (only the first cap are written), or
 * QSIM_EINVAL / QSIM_ERANGE. */
int qsim_plan_make_local(int n, int world, int *pos_io, const int *need, int nneed, int *steps, int cap);
int qsim_plan_canonical_globals(int n, int world, int *pos_io, int *steps, int cap);

#ifdef __cplusplus
}
#endif

#endif /* QSIM_H */
