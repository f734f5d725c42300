// api.cu -- the C-ABI of libqsim (include/qsim.h): validation, the
// logical -> physical qubit map, gate-matrix construction on the host, and
// dispatch to the sm_100a kernels.  No amplitude is ever computed on the
// host: every step of the path runs in the kernels of k_*.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "philox.cuh"
#include "qsim_internal.h"

using namespace qs;

namespace qs {

static std::string g_create_error;

int fail(Handle *h, int code, const std::string &msg)
{
    if (h) h->err = msg;
    else g_create_error = msg;
    return code;
}

int check_cuda(Handle *h, cudaError_t e, const char *what)
{
    if (e == cudaSuccess) return QSIM_OK;
    if (h) h->poisoned = 1;
    return fail(h, QSIM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void ensure_red(Handle *h, size_t doubles)
{
    cudaSetDevice(h->device);
    if (h->red_cap >= doubles) return;
    if (h->d_red) {
        cudaStreamSynchronize(h->stream);
        cudaFree(h->d_red);
    }
    size_t cap = std::max<size_t>(doubles, 1 << 16);
    if (cudaMalloc(&h->d_red, cap * sizeof(double)) != cudaSuccess) {
        h->d_red = nullptr;
        h->red_cap = 0;
        h->poisoned = 1;
        h->err = "cannot allocate reduction workspace";
        return;
    }
    h->red_cap = cap;
}

void ensure_hred(Handle *h, size_t doubles)
{
    cudaSetDevice(h->device);
    if (h->hred_cap >= doubles) return;
    if (h->h_red) cudaFreeHost(h->h_red);
    size_t cap = std::max<size_t>(doubles, 1 << 12);
    if (cudaMallocHost(&h->h_red, cap * sizeof(double)) != cudaSuccess) {
        h->h_red = nullptr;
        h->hred_cap = 0;
        h->poisoned = 1;
        h->err = "cannot allocate pinned host workspace";
        return;
    }
    h->hred_cap = cap;
}

int ensure_scratch(Handle *h)
{
    cudaSetDevice(h->device);
    if (h->scratch) return QSIM_OK;
    cudaError_t e = cudaMalloc(&h->scratch, sizeof(double2) * h->local_dim());
    if (e != cudaSuccess) {
        // recoverable: callers fall back to in-place schedules where they have one
        // (a 2^33-amplitude state fills 128 of the B200's 180 GB: no room for a copy)
        h->scratch = nullptr;
        cudaGetLastError();
        return fail(h, QSIM_ENOMEM, "cannot allocate the " + std::to_string(sizeof(double2) * h->local_dim()) +
                                        "-byte scratch shard");
    }
    return QSIM_OK;
}

static cudaEvent_t pool_event(Handle *h)
{
    if (h->ev_used == h->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        h->ev_pool.push_back(e);
    }
    return h->ev_pool[h->ev_used++];
}

void prof_begin(Handle *h)
{
    cudaSetDevice(h->device);   // rank groups may span devices: launch on the member's own
    if (!h->prof_on) return;
    h->pending = pool_event(h);
    cudaEventRecord(h->pending, h->stream);
}

// communication (NCCL / peer copies): timed like a kernel, not counted as one of ours
void prof_end_comm(Handle *h, const char *name, uint64_t bytes)
{
    if (!h->prof_on || !h->pending) return;
    cudaEvent_t b = pool_event(h);
    cudaEventRecord(b, h->stream);
    h->prof.push_back({name, bytes, h->pending, b, 0});
    h->pending = nullptr;
}

void prof_end(Handle *h, const char *name, uint64_t bytes)
{
    h->launches++;
    const uint64_t fp64 = h->prof_fp64;
    h->prof_fp64 = 0;
    if (!h->prof_on || !h->pending) return;
    cudaEvent_t b = pool_event(h);
    cudaEventRecord(b, h->stream);
    h->prof.push_back({name, bytes, h->pending, b, fp64});
    h->pending = nullptr;
}

}  // namespace qs

// ----------------------------------------------------------------- helpers
namespace {

#define QS_CHECK_HANDLE(h)                                                       \
    do {                                                                         \
        if (!(h)) return QSIM_EINVAL;                                            \
        if ((h)->poisoned) return fail((h), QSIM_ESTATE, "handle is poisoned: " + (h)->err); \
    } while (0)

int after_launch(Handle *h, const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return check_cuda(h, e, what);
    if (h->poisoned) return fail(h, QSIM_ECUDA, h->err);
    return QSIM_OK;
}

bool is_local(const Handle *h, int q) { return h->pos[q] < h->nl; }

// 2x2 complex product C = A B (row-major)
void mat_mul(const double2 A[4], const double2 B[4], double2 C[4])
{
    auto mul = [](double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); };
    auto add = [](double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); };
    double2 r[4];
    r[0] = add(mul(A[0], B[0]), mul(A[1], B[2]));
    r[1] = add(mul(A[0], B[1]), mul(A[1], B[3]));
    r[2] = add(mul(A[2], B[0]), mul(A[3], B[2]));
    r[3] = add(mul(A[2], B[1]), mul(A[3], B[3]));
    std::memcpy(C, r, sizeof r);
}

// U_R(t) = (cos -sin; sin cos), U_P1(p) = diag(1, e^{ip}), U_P2(p) = diag(e^{ip}, 1)
// (PAPER.md:542-561).
void mat_ur(double t, double2 U[4])
{
    U[0] = make_double2(std::cos(t), 0); U[1] = make_double2(-std::sin(t), 0);
    U[2] = make_double2(std::sin(t), 0); U[3] = make_double2(std::cos(t), 0);
}
void mat_up1(double p, double2 U[4])
{
    U[0] = make_double2(1, 0); U[1] = make_double2(0, 0);
    U[2] = make_double2(0, 0); U[3] = make_double2(std::cos(p), std::sin(p));
}
void mat_up2(double p, double2 U[4])
{
    U[0] = make_double2(std::cos(p), std::sin(p)); U[1] = make_double2(0, 0);
    U[2] = make_double2(0, 0); U[3] = make_double2(1, 0);
}

int kind_nangles(int kind) { return kind == QSIM_GATE_RP ? 2 : kind == QSIM_GATE_P1 ? 1 : 4; }

// Angle-form matrix (R12-R15), perturbed when sigma > 0.
// the perturbed angles of gate g: ang[s] + sigma z(draw(seed, OPNOISE, g, s)) (R12-R13)
void noisy_angles(const Handle *h, int kind, const double *ang, uint64_t g, double a[4])
{
    for (int s = 0; s < 4; ++s) a[s] = 0.0;
    const int na = kind_nangles(kind);
    for (int s = 0; s < na; ++s) {
        a[s] = ang[s];
        if (h->sigma > 0.0) {
            const u64x2 d = draw(h->noise_seed, QSIM_TAG_OPNOISE, g, (uint32_t)s);
            const double z = std::sqrt(-2.0 * std::log(u01o(d.a))) * std::cos(2.0 * M_PI * u01(d.b));
            a[s] += h->sigma * z;
        }
    }
}

void angle_matrix(const Handle *h, int kind, const double *ang, uint64_t g, double2 U[4])
{
    double a[4];
    noisy_angles(h, kind, ang, g, a);
    double2 A[4], B[4], C[4];
    if (kind == QSIM_GATE_RP) {
        mat_ur(a[0], A); mat_up1(a[1], B); mat_mul(A, B, U);
    } else if (kind == QSIM_GATE_P1) {
        mat_up1(a[0], U);
    } else {
        mat_up2(a[0], A); mat_up1(a[1], B); mat_mul(A, B, C);
        mat_ur(a[2], A); mat_mul(C, A, B);
        mat_up1(a[3], A); mat_mul(B, A, U);
    }
}

// Translate a controlled gate's qubit sets into a local mask/value pair and
// decide whether this rank participates at all (global controls).
bool local_controls(const Handle *h, uint64_t cmask, uint64_t cvals, uint64_t &lm, uint64_t &lv)
{
    lm = 0;
    lv = 0;
    for (int q = 0; q < h->n; ++q) {
        if (!((cmask >> q) & 1)) continue;
        const int p = h->pos[q];
        const uint64_t want = (cvals >> q) & 1;
        if (p < h->nl) {
            lm |= 1ull << p;
            lv |= want << p;
        } else {
            const uint64_t have = ((uint64_t)h->rank >> (p - h->nl)) & 1;
            if (have != want) return false;
        }
    }
    return true;
}

bool is_diag(const double2 U[4]) { return U[1].x == 0 && U[1].y == 0 && U[2].x == 0 && U[2].y == 0; }

// Immediate (unfused) application of a queued op.
void run_op_now(Handle *h, const QOp &op)
{
    qs::run_gate_unfused(h, op);
}

}  // namespace

// The paper's one-sweep-per-gate kernels (k_gates.cu) for one queued op.
void qs::run_gate_unfused(Handle *h, const QOp &op)
{
    if (op.diag) {
        if (op.tpos >= 0) launch_apply_diag(h, op.tpos, op.cmask, op.cval, op.u[0], op.u[3]);
        else if (!(op.u[3].x == 1.0 && op.u[3].y == 0.0)) launch_phase_mask(h, op.cmask, op.cval, op.u[3]);
    } else {
        launch_apply_2x2(h, op.tpos, op.cmask, op.cval, op.u);
    }
}

namespace {

// A member's failure is reported on the handle the caller holds.
int lift(Handle *top, const Ranks &R, int rc)
{
    if (rc == QSIM_OK || R.size() == 1) return rc;
    for (Handle *m : R) {
        if (!m->err.empty()) top->err = m->err;
        if (m->poisoned) top->poisoned = 1;
    }
    return rc;
}

// Core gate application on logical target q with logical controls, on every
// rank of R: a non-diagonal gate on a rank-bit qubit first makes it local
// (dist.cu); then each rank translates the gate to physical local positions
// (controls on rank bits are decided per rank, a diagonal gate on a rank bit
// becomes a constant phase) and queues it; the queue is fused into tile
// passes at the next flush (or run at once when fusion is off / the shard is
// tiny).
int apply_gate(const Ranks &R, uint64_t cmask, uint64_t cvals, int q, const double2 U[4],
               const std::vector<const double2 *> *tabs = nullptr)
{
    if (R[0]->batch_b && (q < R[0]->batch_b || (cmask & ((1ull << R[0]->batch_b) - 1))))
        return fail(R[0], QSIM_EINVAL, "gate on a trajectory-index qubit of a batched handle");
    const int diag = tabs ? 0 : is_diag(U);
    if (!diag && !is_local(R[0], q)) {
        // one sweep per gate (fusion off): the gate reads the partner's shard
        // over peer memory (one kernel, no layout change, no exchange).  With
        // fusion on, q is swapped onto a local bit instead, so this and the
        // following gates on q join fused passes.
        if (!tabs && !R[0]->fuse && dist_remote_gate_available(R)) return dist_remote_gate(R, cmask, cvals, q, U);
        if (int rc = dist_make_local(R, std::vector<int>{q})) return rc;
    }
    for (size_t ri = 0; ri < R.size(); ++ri) {
        Handle *h = R[ri];
        QOp op;
        op.diag = diag;
        for (int k = 0; k < 4; ++k) op.u[k] = U[k];
        if (tabs) op.tab = (*tabs)[ri];
        uint64_t lm, lv;
        if (!local_controls(h, cmask, cvals, lm, lv)) continue;
        op.cmask = lm;
        op.cval = lv;
        const int p = h->pos[q];
        if (p < h->nl) {
            op.tpos = p;
        } else {
            // diagonal gate on a rank bit: a constant phase under the controls
            const int b = (h->rank >> (p - h->nl)) & 1;
            const double2 d = b ? U[3] : U[0];
            if (d.x == 1.0 && d.y == 0.0) continue;
            op.tpos = -1;
            op.u[0] = make_double2(1.0, 0.0);
            op.u[3] = d;
        }
        if ((h->fuse && h->nl >= 9) || op.tab) {
            h->queue.push_back(op);
            if (h->queue.size() >= 4096)
                if (int rc = flush_queue(h)) return rc;
            continue;
        }
        run_op_now(h, op);
        if (int rc = after_launch(h, "gate")) return rc;
    }
    return QSIM_OK;
}

int check_qubit(Handle *h, int q)
{
    if (q < 0 || q >= h->n) return fail(h, QSIM_ERANGE, "qubit " + std::to_string(q) + " outside [0, n)");
    return QSIM_OK;
}

// strict mode (qsim_set_strict): max |(U U^dagger - I)_rc| <= 1e-12, the
// paper's gates being unitary
int check_unitary(Handle *h, const double2 U[4])
{
    if (!h->strict) return QSIM_OK;
    double e = 0.0;
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) {
            // sum_k U[r][k] conj(U[c][k])
            double re = 0.0, im = 0.0;
            for (int k = 0; k < 2; ++k) {
                const double2 a = U[2 * r + k], b = U[2 * c + k];
                re += a.x * b.x + a.y * b.y;
                im += a.y * b.x - a.x * b.y;
            }
            if (r == c) re -= 1.0;
            e = std::max(e, std::hypot(re, im));
        }
    if (!(e <= 1e-12)) return fail(h, QSIM_ENONUNITARY, "matrix is not unitary: max |U U^dagger - I| = " + std::to_string(e));
    return QSIM_OK;
}

int check_ctrl(Handle *h, uint64_t cmask, uint64_t cvals, int q)
{
    if (h->n < 64 && (cmask >> h->n)) return fail(h, QSIM_ERANGE, "control mask has qubits >= n");
    if ((cmask >> q) & 1) return fail(h, QSIM_EINVAL, "target qubit is also a control");
    if (cvals & ~cmask) return fail(h, QSIM_EINVAL, "ctrl_vals has bits outside ctrl_mask");
    return QSIM_OK;
}

// Build a TilePass from a tile (tile bit -> input local position) and a full
// local permutation perm (input position -> output position).
TilePass make_pass(const Handle *h, const std::vector<int> &tile_pos, const std::vector<int> &perm)
{
    TilePass tp;
    std::memset(&tp, 0, sizeof tp);
    tp.tbits = (int)tile_pos.size();
    std::vector<char> in_tile(h->nl, 0);
    for (int b = 0; b < tp.tbits; ++b) {
        tp.in_pos[b] = tile_pos[b];
        tp.out_pos[b] = perm[tile_pos[b]];
        in_tile[tile_pos[b]] = 1;
    }
    tp.nfix = 0;
    for (int p = 0; p < h->nl; ++p) {
        if (in_tile[p]) continue;
        tp.fin_pos[tp.nfix] = p;
        tp.fout_pos[tp.nfix] = perm[p];
        tp.nfix++;
    }
    tp.scale = 1.0;
    return tp;
}


// Fused H / QFT on the wires [lo, lo+m) (logical).  qft = 0: Hadamard transform.
//
// Wires are cut into G blocks of <= amax consecutive wires; pass g applies
// every gate of block g (see k_tile.cu / k_tma.cu).  A pass reads tiles of
// 2^12 amplitudes: the block's wires + the lowest other positions
// ("passive", so a tile moves in runs of >= 2^(12-a) contiguous amplitudes).
//
// Single GPU, QFT: the closing swaps are folded into the stores with a
// block-move layout (no extra pass).  Invariant before pass g (wires
// 0..a0-1 done): positions [s0, s0+a0) hold wires 0..a0-1 in final order,
// positions [s0+a0, s0+m) hold wires a0..m-1 descending (wire a0 on top;
// s0 = lowest position of the range).  Pass g writes its block to
// [s0+a0, s0+a0+a) ascending and shifts the rest up by a, so after the last
// pass wire w sits at s0+w, which is where logical qubit lo+m-1-w lived:
// the swapped labels land exactly on the canonical layout.  Every position
// run stays contiguous, so each pass is one <= 5-D TMA box per tile.
// Several ranks: before each pass the block's wires are made local (shard
// exchanges), passes run in place, and the closing swaps are a relabelling.
// The QFT circuit with per-gate data (operational error, PAPER.md:540-569;
// approximate QFT) in the wire numbering of fused_range:
// H[w] = the matrix of H(lo+w), phi[i][k] / e[i][k] (i < k) = the angle /
// phase factor of the R between wires i and k (0 when the gate is absent).
struct GenCircuit {
    int m;
    std::vector<double> Hr;   // 4 m: H(lo+w) = Hr[w] diag(1, e^{i hph[w]})
    std::vector<double> hph;  // m
    std::vector<double> phi;  // m m
    std::vector<double2> e;   // m m
};

constexpr int kGenInfeasible = 1000;   // dry run: a pass the generalised kernel cannot take

// One fused QFT / H block of an in-process rank group whose wires gw (block
// indices, 1 or 2 of them) sit on rank bits: k_qft13 in rank-group mode on
// every member -- each takes the tiles whose split bits equal its own rank
// bits, lands the tile's rows from the 2^ng shards that hold them (peer
// memory over NVLink between GPUs) and stores every amplitude back in place
// into the shard its global bits name.  The paper's pairing rule (rows R_j
// and R_{2^P+j} meet on one processor) is met inside the
// tile instead of by moving half of each shard first.  Returns 1 (nothing
// launched) when the geometry does not fit.
int rank_group_pass(const Ranks &R, const std::vector<int> &wp, int a0, int a, const std::vector<int> &gw, int qft,
                    int inverse)
{
    Handle *h0 = R[0];
    const int nl = h0->nl, ng = (int)gw.size();
    // tile: block wires (tile bits 0..a-1) + the lowest 13 - a local positions
    std::vector<int> tpos;
    std::vector<char> in_t(nl, 0);
    for (int u = 0; u < a; ++u) {
        const int p = wp[a0 + u];
        tpos.push_back(p);
        if (p < nl) in_t[p] = 1;
    }
    for (int p = 0; p < nl && (int)tpos.size() < kTile13Bits; ++p)
        if (!in_t[p]) { tpos.push_back(p); in_t[p] = 1; }
    if ((int)tpos.size() != kTile13Bits) return 1;
    std::vector<int> gbits(gw);
    std::sort(gbits.begin(), gbits.end(), [&](int x, int y) { return wp[a0 + x] < wp[a0 + y]; });
    // one process per GPU: the peers' shards through CUDA IPC (collective; all
    // ranks agree on availability); an in-process group addresses them directly
    std::vector<double2 *> world_shards;
    const bool world_mode = R.size() == 1;
    if (world_mode) {
        if (int rc = flush_queue(h0)) return rc;
        if (int rc = dist_world_shards(h0, world_shards)) return rc;   // 1: no IPC, the caller exchanges
    }
    std::vector<Qft13Desc> ds(R.size());
    for (size_t r = 0; r < R.size(); ++r) {
        Handle *h = R[r];
        Qft13Desc &d = ds[r];
        std::memset(&d, 0, sizeof d);
        d.a = a;
        for (int b = 0; b < kTile13Bits; ++b) {
            d.in_pos[b] = tpos[b];
            d.out_pos[b] = tpos[b] < nl ? tpos[b] : -1;
        }
        for (int p = 0; p < nl; ++p)
            if (!in_t[p]) {
                d.fin_pos[d.nfix] = p;
                d.fout_pos[d.nfix] = p;
                d.nfix++;
            }
        if (d.nfix < ng) return 1;
        d.W = a0 + a;
        d.inverse = inverse;
        d.hadamard_only = !qft;
        d.scale = std::ldexp(1.0, -(a / 2));
        if (a & 1) d.scale *= M_SQRT1_2;
        if (qft) {
            for (int i = 0; i < a0; ++i) {
                const int p = wp[i];
                if (p >= nl) { d.y_const += (uint64_t)((h->rank >> (p - nl)) & 1) << i; continue; }
                int b = -1;
                for (int t = 0; t < kTile13Bits; ++t) if (d.in_pos[t] == p) b = t;
                if (b >= 0) { d.et_bit[d.n_et] = b; d.et_w[d.n_et] = i; d.n_et++; }
                else {
                    int f = -1;
                    for (int t = 0; t < d.nfix; ++t) if (d.fin_pos[t] == p) f = t;
                    d.ef_bit[d.n_ef] = f; d.ef_w[d.n_ef] = i; d.n_ef++;
                }
            }
        }
        d.ng = ng;
        for (int i = 0; i < ng; ++i) {
            d.gbit[i] = gbits[i];
            d.split_fix[i] = d.nfix - ng + i;
            const int rb = wp[a0 + gbits[i]] - nl;
            d.split_val |= (uint64_t)((h->rank >> rb) & 1) << i;
        }
        for (int c = 0; c < (1 << ng); ++c) {
            int rr = h->rank;
            for (int i = 0; i < ng; ++i) {
                const int rb = wp[a0 + gbits[i]] - nl;
                rr = (rr & ~(1 << rb)) | (((c >> i) & 1) << rb);
            }
            d.gbase[c] = world_shards.empty() ? R[rr]->psi : world_shards[rr];
        }
    }
    // every member's earlier work on its shard is done before anyone reads it
    const size_t P = R.size();
    std::vector<cudaEvent_t> ev(P);
    auto all_wait = [&]() {
        for (size_t i = 0; i < P; ++i) {
            cudaSetDevice(R[i]->device);
            cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
            cudaEventRecord(ev[i], R[i]->stream);
        }
        for (size_t i = 0; i < P; ++i) {
            cudaSetDevice(R[i]->device);
            for (size_t j = 0; j < P; ++j) cudaStreamWaitEvent(R[i]->stream, ev[j], 0);
        }
        for (size_t i = 0; i < P; ++i) {
            cudaSetDevice(R[i]->device);
            cudaEventDestroy(ev[i]);
        }
    };
    if (world_mode) {
        // every rank's earlier work is done before anyone touches its shard;
        // afterwards no rank moves on while a peer may still write into it
        if (int rc = dist_world_barrier(h0)) return rc;
        if (!launch_qft13(h0, ds[0], h0->psi, h0->psi))
            return fail(h0, QSIM_ECUDA, "rank-group pass geometry rejected after the shards were mapped");
        if (int rc = after_launch(h0, "rank-group pass")) return rc;
        return dist_world_barrier(h0);
    }
    for (Handle *h : R) {
        cudaSetDevice(h->device);
        if (int rc = flush_queue(h)) return rc;
    }
    all_wait();
    for (size_t r = 0; r < P; ++r) {
        if (!launch_qft13(R[r], ds[r], R[r]->psi, R[r]->psi)) {
            if (r == 0) return 1;
            return fail(R[r], QSIM_ECUDA, "rank-group pass geometry differs between members");
        }
        if (int rc = after_launch(R[r], "rank-group pass")) return rc;
    }
    all_wait();   // a member's later work waits for every member that wrote into its shard
    return QSIM_OK;
}

int fused_range(const Ranks &R, int lo, int m, int qft, int inverse, const GenCircuit *gc = nullptr,
                bool dry = false, bool even = false)
{
    // default 8: a 2^12 tile then carries >= 4 passive bits (>= 256-byte runs); measured
    // (tools/probe_amax.py) against 7 (>= 512-byte runs) and 9 (128-byte runs): 8 needs
    // fewer passes for most register sizes (n = 29: 4 instead of 5, a 22-wire range 3
    // instead of 4) and is as fast per pass -- the n = 28 QFT runs 8,7,7,6 in 5.45 ms
    // (7,7,7,7: 5.49 ms); 10 wires would leave 64-byte runs (~70% of peak)
    // (the generalised kernel, FP64-heavier per wire, stays at 7: its 8-wire passes ran slower)
    static const int amax_env = getenv("QSIM_QFT_AMAX") ? atoi(getenv("QSIM_QFT_AMAX")) : 0;
    const int amax_def = amax_env > 0 ? amax_env : (gc ? 7 : 8);
    const int amax = amax_def < 1 ? 1 : (amax_def > 10 ? 10 : amax_def);
    Handle *h0 = R[0];
    const int G = (m + amax - 1) / amax;
    std::vector<int> gsize(G, m / G);
    for (int g = 0; g < m % G; ++g) gsize[g]++;
    // the block-move layout writes out of place whenever a pass moves fixed
    // bits: without room for a scratch shard the passes run in place and the
    // closing swaps become a relabel (as on several ranks)
    static const bool no_moves = getenv("QSIM_NO_BLOCK_MOVES") != nullptr;   // measurement knob
    const bool block_moves = qft && h0->world == 1 && !no_moves && ensure_scratch(h0) == QSIM_OK;
    if (block_moves && G > 2 && amax == 8 && !gc && !even) {
        // measured per-pass efficiency (tools/probe_blocks.sh): 8- and 6-wire
        // passes stream best, 7 a little worse, <= 5 and a last block of 8
        // worse: 8,...,8 then the remainder r of the last two blocks as (8, r-8)
        // when r-8 >= 6, else split evenly -- n = 28: 8,8,6,6 (5.43 ms vs
        // 5.45 for 8,7,7,6), n = 29: 8,8,7,6, n = 30: 8,8,8,6
        for (int g = 0; g < G - 2; ++g) gsize[g] = 8;
        const int r = m - 8 * (G - 2);
        if (r - 8 >= 6) {
            gsize[G - 2] = 8;
            gsize[G - 1] = r - 8;
        } else {
            gsize[G - 2] = (r + 1) / 2;
            gsize[G - 1] = r / 2;
        }
    } else if (block_moves && G > 1 && gsize[0] < amax && !even) {
        // the first block lands on the lowest positions; with >= 7 wires its
        // last register window stays clear of the 3 lowest, so the store keeps
        // 128-byte thread runs and the pass fits the specialised kernel
        // (k_qft_tma) -- put the full amax there, spread the rest evenly
        gsize[0] = amax;
        const int rest = m - amax, G1 = G - 1;
        for (int g = 1; g < G; ++g) gsize[g] = rest / G1 + (g - 1 < rest % G1 ? 1 : 0);
    }
    // 2^13-amplitude tiles (k_qft13): one more passive bit per pass, so blocks
    // of 9-10 wires keep 128-256-byte runs and the register needs
    // ceil(m / 10) passes (n = 28: 10, 9, 9 -- three passes instead of four;
    // measured per pass in profiles/r2_qft_passes.md).  The first block may
    // take 10 wires: with block moves it writes one contiguous run per tile.
    static const bool no13 = getenv("QSIM_NO_QFT13") != nullptr;   // measurement knob
    const bool force13 = getenv("QSIM_FORCE_QFT13") != nullptr;   // test / measurement knob (read per call)
    // only where it saves a pass: a 12-bit pass of <= 8 wires streams faster
    // (6.2-6.5 vs 5.4-6.1 TB/s), so ceil(m/10) must beat ceil(m/8)
    // (m = 31: 8,8,8,7 on 12-bit tiles 43.6 ms vs 48.9 ms on 13-bit tiles)
    const bool use13 = !gc && !no13 && h0->nl >= kTile13Bits + 2 && m >= 10 &&
                       (force13 || (m + 9) / 10 < (m + 7) / 8);
    if (use13 && !even) {
        const int G13 = (m + 9) / 10;
        gsize.assign(G13, 0);
        gsize[0] = std::min(10, m - 5 * (G13 - 1));
        const int rest = m - gsize[0], G1 = G13 - 1;
        for (int g = 1; g < G13; ++g) gsize[g] = rest / G1 + (g - 1 < rest % G1 ? 1 : 0);
    }
    if (const char *bl = getenv("QSIM_QFT_BLOCKS")) {   // measurement knob: explicit block sizes (tools/probe_blocks.sh)
        std::vector<int> v;
        int s = 0;
        for (const char *c = bl; *c;) {
            const int x = atoi(c);
            v.push_back(x);
            s += x;
            while (*c && *c != ',') ++c;
            if (*c) ++c;
        }
        bool ok = s == m && !v.empty();
        for (int x : v) ok &= x >= 1 && x <= 10;
        if (ok) gsize = v;
    }
    if (block_moves) {
        if (int rc = dist_canonicalize(R)) return rc;
    } else {
        if (int rc = flush_all(R)) return rc;
    }
    const int nl = h0->nl;
    const int s0 = h0->n - lo - m;         // lowest position of the range (canonical)
    std::vector<int> wp(m);                // current position of wire w (same on every rank)
    for (int w = 0; w < m; ++w) wp[w] = h0->pos[lo + w];
    // Free intermediate layouts on one GPU ("H passes"): every
    // pass but the last writes its tile out of place to the lowest 13
    // positions (one contiguous run per tile) and parks the next block's wires
    // on the top positions; the last pass puts every bit where it ends.  H
    // (every wire ends where it started: the in-place passes had 128-byte rows
    // on both sides for the top block, and the lowest block stayed on the
    // 12-bit kernel) and the QFT of a sub-register above position 0 (its block
    // moves wrote 128-byte rows, the passives being the other qubits).  The
    // plan is simulated first; a plan whose passes cannot all have
    // conflict-free landing reads and coalesced stores keeps the old one.
    const int Gn = (int)gsize.size();
    static const bool no_hflex = getenv("QSIM_NO_HFLEX") != nullptr;   // measurement knob
    static const bool no_qflex = getenv("QSIM_NO_QFLEX") != nullptr;   // measurement knob
    bool hflex = (qft ? block_moves && s0 > 0 && !no_qflex : !no_hflex) && !gc && !dry && use13 && R.size() == 1 &&
                 h0->world == 1 && Gn >= 2;
    for (int a : gsize) hflex &= a >= 5 && a <= 10;
    for (int w = 0; w < m && hflex; ++w) hflex &= wp[w] < nl;
    std::vector<std::vector<int>> hf_tpos(Gn), hf_perm(Gn);
    std::vector<int> hat(nl), fin_of(nl);  // hat[p]: start position of the bit now at p; fin_of: its end
    for (int p = 0; p < nl; ++p) hat[p] = fin_of[p] = p;
    if (hflex && qft)
        for (int w = 0; w < m; ++w) fin_of[wp[w]] = s0 + w;   // the closing swaps, as the block moves
    if (hflex) {
        std::vector<int> blk_of(nl, -1);   // start position -> block of its wire
        for (int g = 0, b0 = 0; g < Gn; b0 += gsize[g], ++g)
            for (int u = 0; u < gsize[g]; ++u) blk_of[wp[b0 + u]] = g;
        std::vector<int> swp(wp), shat(hat);
        for (int g = 0, b0 = 0; g < Gn && hflex; b0 += gsize[g], ++g) {
            const int a = gsize[g];
            const bool last = g + 1 == Gn;
            auto fin = [&](int p) { return fin_of[shat[p]]; };
            std::vector<char> is_act(nl, 0);
            std::vector<int> act;
            for (int u = 0; u < a; ++u) { act.push_back(swp[b0 + u]); is_act[swp[b0 + u]] = 1; }
            std::vector<int> pas;
            for (int p = 0; p < nl && (int)pas.size() < kTile13Bits - a; ++p)
                if (!is_act[p]) pas.push_back(p);
            std::vector<int> sorted(act);
            sorted.insert(sorted.end(), pas.begin(), pas.end());
            std::sort(sorted.begin(), sorted.end());
            auto rank = [&](int p) { return (int)(std::lower_bound(sorted.begin(), sorted.end(), p) - sorted.begin()); };
            // window 0 (tile bits 0..4).  The QFT: the block's first five wires
            // (its phases fix the order).  H (any order): the 5 highest-ranked
            // actives in a non-final pass, the 5 with the lowest final positions
            // in the last one (its stores then run over the lowest outputs from
            // the lanes), the wire that ends on position 0 in window 1
            // (neighbouring pairs per thread: 32-byte stores)
            std::vector<int> ord(act);
            if (!qft && last) {
                std::sort(ord.begin(), ord.end(), [&](int x, int y) { return fin(x) < fin(y); });
                if (a >= 6 && fin(ord[0]) == 0) {
                    const int z = ord[0];
                    ord.erase(ord.begin());
                    ord.insert(ord.begin() + 5, z);
                }
            } else if (!qft) {
                std::sort(ord.begin(), ord.end(), [&](int x, int y) { return x > y; });
            }
            for (int i = 0; i < 5; ++i) hflex &= rank(ord[i]) >= 5;   // landing reads stay conflict-free
            std::vector<int> tpos(ord);
            tpos.insert(tpos.end(), pas.begin(), pas.end());
            std::vector<int> perm(nl, -1);
            if (last) {
                for (int p = 0; p < nl; ++p) perm[p] = fin(p);
                // the QFT: the last window's wires off the tile's five lowest
                // output positions (those are the lanes' for coalesced stores)
                std::vector<std::pair<int, int>> outs;   // (output position, window-1 bit?)
                for (int b = 0; b < kTile13Bits; ++b) outs.push_back({perm[tpos[b]], b >= a - 5 && b < a});
                std::sort(outs.begin(), outs.end());
                for (int i = 0; i < 5 && qft; ++i) hflex &= !outs[i].second;
            } else {
                // outputs 0..12: [tile bits that stay thread bits in map 1, by
                // final position] [window-1 bits] [later blocks' wires]; then the
                // fixed bits, the next block last (lowest final position on top)
                std::vector<char> in_t(nl, 0), in_w1(nl, 0);
                for (int p : tpos) in_t[p] = 1;
                for (int b = a - 5; b < a; ++b) in_w1[tpos[b]] = 1;
                std::vector<int> s0v, s1, s2, f0, f1;
                for (int p : tpos) {
                    if (blk_of[shat[p]] > g) s2.push_back(p);
                    else if (in_w1[p]) s1.push_back(p);
                    else s0v.push_back(p);
                }
                for (int p = 0; p < nl; ++p)
                    if (!in_t[p]) (blk_of[shat[p]] == g + 1 ? f1 : f0).push_back(p);
                auto up = [&](int x, int y) { return fin(x) < fin(y); };
                auto down = [&](int x, int y) { return fin(x) > fin(y); };
                std::sort(s0v.begin(), s0v.end(), up);
                std::sort(s1.begin(), s1.end(), up);
                std::sort(s2.begin(), s2.end(), down);
                // H: the final block's wires with the lowest final positions on
                // top (they are that pass's window 0); otherwise a block keeps
                // its order (tiles running at the same time then write
                // neighbouring regions, as the QFT's block moves do)
                if (!qft && g + 2 == Gn) std::sort(f1.begin(), f1.end(), down);
                int q = 0;
                if (!qft && !s1.empty()) { perm[s1[0]] = q++; s1.erase(s1.begin()); }   // H: pair stores
                for (int p : s0v) perm[p] = q++;
                hflex &= q >= 5;   // the lanes' output positions are not window bits
                for (auto *v : {&s1, &s2, &f0, &f1})
                    for (int p : *v) perm[p] = q++;
            }
            hf_tpos[g] = tpos;
            hf_perm[g] = perm;
            for (int w = 0; w < m; ++w) swp[w] = perm[swp[w]];
            std::vector<int> nh(nl);
            for (int p = 0; p < nl; ++p) nh[perm[p]] = shat[p];
            shat = nh;
        }
        if (hflex && ensure_scratch(h0) != QSIM_OK) hflex = false;
    }
    bool hflex_off = false;                // a planned pass fell back: in place from there on
    int a0 = 0;
    for (int g = 0; g < (int)gsize.size(); ++g) {
        const int a = gsize[g];
        const bool hf = hflex && !hflex_off;
        std::vector<int> act;
        for (int u = 0; u < a; ++u) act.push_back(lo + a0 + u);
        if (h0->world > 1) {
            // in-process rank groups: a block with one or two wires on rank bits
            // runs as one rank-group pass over peer memory (the exchange fused
            // into the pass, nothing moves beforehand); otherwise the block's
            // wires are made local by shard exchanges first
            static const bool no_rg = getenv("QSIM_NO_RANK_GROUP_PASS") != nullptr;   // measurement knob
            std::vector<int> gw;
            for (int u = 0; u < a; ++u)
                if (wp[a0 + u] >= h0->nl) gw.push_back(u);
            if (!no_rg && use13 && !dry && !gw.empty() && gw.size() <= 2 && a >= 5 && a <= 10 &&
                a - (int)gw.size() <= h0->nl) {
                const int rc = rank_group_pass(R, wp, a0, a, gw, qft, inverse);
                if (rc == QSIM_OK) {
                    a0 += a;
                    continue;
                }
                if (rc != 1) return rc;   // 1: geometry not supported, fall through
            }
            if (int rc = dist_make_local(R, act)) return rc;
            for (int w = 0; w < m; ++w) wp[w] = h0->pos[lo + w];
        }
        // output permutation of the local positions (block moves)
        std::vector<int> perm13(nl);
        for (int p = 0; p < nl; ++p) perm13[p] = p;
        if (block_moves && !hflex) {
            for (int w = a0 + a; w < m; ++w) perm13[wp[w]] = wp[w] + a;
            for (int u = 0; u < a; ++u) perm13[wp[a0 + u]] = s0 + a0 + u;
        }
        // in place (no block moves), a block on the lowest positions would put
        // them in the last register window: 512-byte runs per thread, one
        // 16-byte store per lane per run -- that pass stays on the 12-bit kernel
        bool low_block = false;
        for (int u = 0; u < a; ++u) low_block |= !block_moves && !hf && wp[a0 + u] < kTile13Bits - a + 5;
        if (use13 && a >= 5 && a <= 10 && !dry && !low_block) {
            // the 13-bit pass: active wires + the lowest 13 - a other positions
            std::vector<int> tpos;
            std::vector<char> in13(nl, 0);
            for (int u = 0; u < a; ++u) { tpos.push_back(wp[a0 + u]); in13[wp[a0 + u]] = 1; }
            for (int p = 0; p < nl && (int)tpos.size() < kTile13Bits; ++p)
                if (!in13[p]) { tpos.push_back(p); in13[p] = 1; }
            if (hf) {   // the planned H pass (same tile, windows and output order chosen above)
                tpos = hf_tpos[g];
                perm13 = hf_perm[g];
            }
            bool moved13 = false;
            for (int p = 0; p < nl; ++p) moved13 |= !in13[p] && perm13[p] != p;
            bool ok13 = true;
            for (Handle *h : R) {
                Qft13Desc d;
                std::memset(&d, 0, sizeof d);
                d.a = a;
                for (int b = 0; b < kTile13Bits; ++b) {
                    d.in_pos[b] = tpos[b];
                    d.out_pos[b] = perm13[tpos[b]];
                }
                for (int p = 0; p < nl; ++p)
                    if (!in13[p]) {
                        d.fin_pos[d.nfix] = p;
                        d.fout_pos[d.nfix] = perm13[p];
                        d.nfix++;
                    }
                d.W = a0 + a;
                d.inverse = inverse;
                d.hadamard_only = !qft;
                d.scale = std::ldexp(1.0, -(a / 2));
                if (a & 1) d.scale *= M_SQRT1_2;
                if (qft) {
                    for (int i = 0; i < a0; ++i) {
                        const int p = wp[i];
                        if (p >= nl) { d.y_const += (uint64_t)((h->rank >> (p - nl)) & 1) << i; continue; }
                        int b = -1;
                        for (int t = 0; t < kTile13Bits; ++t) if (d.in_pos[t] == p) b = t;
                        if (b >= 0) { d.et_bit[d.n_et] = b; d.et_w[d.n_et] = i; d.n_et++; }
                        else {
                            int f = -1;
                            for (int t = 0; t < d.nfix; ++t) if (d.fin_pos[t] == p) f = t;
                            d.ef_bit[d.n_ef] = f; d.ef_w[d.n_ef] = i; d.n_ef++;
                        }
                    }
                }
                double2 *out = h->psi;
                if (moved13) {
                    if (ensure_scratch(h)) return QSIM_ENOMEM;
                    out = h->scratch;
                }
                if (!launch_qft13(h, d, h->psi, out)) {
                    if (h != R[0]) return fail(h, QSIM_ECUDA, "13-bit QFT pass geometry differs between ranks");
                    ok13 = false;
                    break;
                }
                if (moved13) swap_buffers(h);
                if (int rc = after_launch(h, "fused tile pass (13)")) return rc;
            }
            if (ok13) {
                for (int w = 0; w < m; ++w)
                    if (wp[w] < nl) wp[w] = perm13[wp[w]];
                if (hf) {
                    std::vector<int> nh(nl);
                    for (int p = 0; p < nl; ++p) nh[perm13[p]] = hat[p];
                    hat = nh;
                }
                a0 += a;
                continue;
            }
        }
        if (hf) hflex_off = true;   // from here on in place on the current layout
        // tile: active wires (tile bits 0..a-1) + passive low positions
        std::vector<int> tile_pos;
        std::vector<char> in_tile(nl, 0);
        for (int u = 0; u < a; ++u) {
            tile_pos.push_back(wp[a0 + u]);
            in_tile[wp[a0 + u]] = 1;
        }
        const int want = std::min(kTileMaxBits, nl);
        for (int p = 0; p < nl && (int)tile_pos.size() < want; ++p)
            if (!in_tile[p]) { tile_pos.push_back(p); in_tile[p] = 1; }
        // output permutation of the local positions
        std::vector<int> perm(nl);
        for (int p = 0; p < nl; ++p) perm[p] = p;
        if (block_moves && !hflex) {
            for (int w = a0 + a; w < m; ++w) perm[wp[w]] = wp[w] + a;   // rest block moves up
            for (int u = 0; u < a; ++u) perm[wp[a0 + u]] = s0 + a0 + u;  // block to final spots
        }
        bool moved_fixed = false;
        for (int p = 0; p < nl; ++p) moved_fixed |= !in_tile[p] && perm[p] != p;
        for (Handle *h : R) {
            TilePass tp = make_pass(h, tile_pos, perm);
            tp.a = a;
            tp.inverse = inverse;
            tp.hadamard_only = !qft;
            tp.scale = std::ldexp(1.0, -(a / 2));
            if (a & 1) tp.scale *= M_SQRT1_2;
            tp.W = a0 + a;
            tp.n_et = tp.n_ef = 0;
            tp.y_const = 0;
            if (qft) {
                for (int i = 0; i < a0; ++i) {
                    const int p = wp[i];
                    if (p >= nl) {   // an earlier wire on a rank bit: constant for this rank
                        tp.y_const += (uint64_t)((h->rank >> (p - nl)) & 1) << i;
                        continue;
                    }
                    int b = -1;
                    for (int t = 0; t < tp.tbits; ++t) if (tp.in_pos[t] == p) b = t;
                    if (b >= 0) { tp.et_bit[tp.n_et] = b; tp.et_w[tp.n_et] = i; tp.n_et++; }
                    else {
                        int f = -1;
                        for (int t = 0; t < tp.nfix; ++t) if (tp.fin_pos[t] == p) f = t;
                        tp.ef_bit[tp.n_ef] = f; tp.ef_w[tp.n_ef] = i; tp.n_ef++;
                    }
                }
            }
            plan_tile_maps(tp);
            if (gc) {
                if (dry) {
                    if (!qft_gen_feasible(h, tp)) return kGenInfeasible;
                    continue;
                }
                QftGen gg;
                std::memset(&gg, 0, sizeof gg);
                for (int u = 0; u < a; ++u) {
                    const int w = a0 + u;
                    for (int k = 0; k < 4; ++k) gg.Hr[u][k] = gc->Hr[4 * w + k];
                    gg.hph[u] = gc->hph[w];
                    for (int u2 = 0; u2 < u; ++u2) gg.ein[u][u2] = gc->e[(a0 + u2) * m + w];
                    for (int i = 0; i < a0; ++i) gg.phe[u][i] = gc->phi[i * m + w];
                }
                double2 *out = h->psi;
                if (moved_fixed) {
                    if (ensure_scratch(h)) return QSIM_ENOMEM;
                    out = h->scratch;
                }
                if (!launch_qft_gen_tma(h, tp, gg, h->psi, out))
                    return fail(h, QSIM_ECUDA, "generalised QFT pass geometry changed after the dry run");
                if (moved_fixed) swap_buffers(h);
            } else if (moved_fixed) {
                if (ensure_scratch(h)) return QSIM_ENOMEM;
                launch_tile_pass(h, tp, h->psi, h->scratch);
                swap_buffers(h);
            } else {
                launch_tile_pass(h, tp, h->psi, h->psi);
            }
            if (int rc = after_launch(h, "fused tile pass")) return rc;
        }
        for (int w = 0; w < m; ++w)
            if (wp[w] < nl) wp[w] = perm[wp[w]];
        a0 += a;
    }
    if (hflex) {
        // a plan that fell back part-way: one permutation pass puts every bit back
        std::vector<int> back(nl);
        bool ident = true;
        for (int p = 0; p < nl; ++p) { back[p] = fin_of[hat[p]]; ident &= back[p] == p; }
        if (!ident) permute_local(h0, back);
    }
    if (qft && !block_moves && !dry) {
        // closing swaps as a relabelling of the logical -> physical map (not in a
        // dry run: fused_qft_gen calls it once or twice before the real pass)
        for (Handle *h : R)
            for (int t = 0; t < m / 2; ++t) std::swap(h->pos[lo + t], h->pos[lo + m - 1 - t]);
    }
    return QSIM_OK;
}

}  // namespace

// Local bit permutation pass: new position of old local position p is perm[p].
void qs::permute_local(Handle *h, const std::vector<int> &perm)
{
    bool ident = true;
    for (int p = 0; p < h->nl; ++p) ident &= perm[p] == p;
    if (ident) return;
    if (h->nl < 9 || ensure_scratch(h) != QSIM_OK) {
        // tiny shards, or no room for an out-of-place pass: a sequence of
        // in-place position swaps
        std::vector<int> cur(h->nl);   // cur[p] = where old position p's bit currently is
        for (int p = 0; p < h->nl; ++p) cur[p] = p;
        std::vector<int> at(h->nl);    // at[x] = old position whose bit sits at x
        for (int p = 0; p < h->nl; ++p) at[p] = p;
        for (int p = 0; p < h->nl; ++p) {
            const int want = perm[p];
            const int now = cur[p];
            if (now == want) continue;
            launch_swap_local(h, now, want);
            const int other = at[want];
            at[want] = p; at[now] = other;
            cur[p] = want; cur[other] = now;
        }
        return;
    }
    // tile = old low positions + the old positions that land on new low positions
    std::vector<int> tile;
    std::vector<char> used(h->nl, 0);
    auto add = [&](int p) { if (!used[p] && (int)tile.size() < kTileMaxBits - 2) { used[p] = 1; tile.push_back(p); } };
    std::vector<int> inv(h->nl);
    for (int p = 0; p < h->nl; ++p) inv[perm[p]] = p;
    for (int k = 0; k < 5 && k < h->nl; ++k) { add(k); add(inv[k]); }
    for (int k = 5; (int)tile.size() < 10 && k < h->nl; ++k) { add(k); }
    TilePass tp = make_pass(h, tile, perm);
    tp.a = 0;
    plan_tile_maps(tp);
    launch_tile_pass(h, tp, h->psi, h->scratch);
    swap_buffers(h);
}

// =================================================================== C-ABI
extern "C" {

uint64_t qsim_memory_bytes(int n) { return (n < 0 || n > 59) ? 0 : (uint64_t)1 << (n + 4); }

const char *qsim_last_error(const qsim_t *h) { return h ? h->err.c_str() : g_create_error.c_str(); }

uint64_t qsim_launch_count(const qsim_t *h)
{
    if (!h) return 0;
    uint64_t s = h->launches;
    for (const Handle *m : h->members) s += m->launches;
    return s;
}

void qsim_philox_draw(uint64_t seed, uint32_t tag, uint64_t i, uint32_t j, uint64_t out[2])
{
    const u64x2 d = draw(seed, tag, i, j);
    out[0] = d.a;
    out[1] = d.b;
}

void qsim_philox_draws(uint64_t seed, uint32_t tag, uint64_t i0, uint64_t count, uint32_t j, uint64_t *out)
{
    if (!out) return;
    for (uint64_t k = 0; k < count; ++k) {
        const u64x2 d = draw(seed, tag, i0 + k, j);
        out[2 * k] = d.a;
        out[2 * k + 1] = d.b;
    }
}

static int create_common(int n, int world, int rank, int device, qsim_t **out)
{
    *out = nullptr;
    if (n < 1 || n > kMaxQubits) return fail(nullptr, QSIM_ERANGE, "n must be in [1, 40]");
    if (world < 1 || (world & (world - 1))) return fail(nullptr, QSIM_EINVAL, "world must be a power of two");
    int kg = 0;
    while ((1 << kg) < world) ++kg;
    if (n - kg < 1) return fail(nullptr, QSIM_ERANGE, "2^n must be >= 2 * world");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, QSIM_ENODEV, "no CUDA device (libqsim has no CPU path)");
    }
    if (device < 0) cudaGetDevice(&device);
    if (device >= ndev) return fail(nullptr, QSIM_ENODEV, "device index out of range");
    cudaSetDevice(device);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    if (prop.major != 10) return fail(nullptr, QSIM_ENODEV, std::string("libqsim is built for sm_100a; device is ") + prop.name);
    qsim_t *h = new qsim_t();
    h->n = n;
    h->world = world;
    h->rank = rank;
    h->kglob = kg;
    h->nl = n - kg;
    h->device = device;
    h->num_sms = prop.multiProcessorCount;
    for (int q = 0; q < n; ++q) h->pos[q] = n - 1 - q;
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete h;
        return fail(nullptr, QSIM_ECUDA, "cannot create stream");
    }
    const size_t bytes = sizeof(double2) * h->local_dim();
    if (cudaMalloc(&h->psi, bytes) != cudaSuccess) {
        cudaGetLastError();
        cudaStreamDestroy(h->stream);
        delete h;
        return fail(nullptr, QSIM_ENOMEM, "cannot allocate " + std::to_string(bytes) +
                                               " bytes of HBM for the state shard (2^(n+4) bytes per state)");
    }
    ensure_red(h, 1 << 16);
    ensure_hred(h, 1 << 12);
    // |0...0>
    launch_zero(h);
    if (rank == 0) launch_set_one(h, 0);
    int rc = after_launch(h, "init");
    if (rc) {
        qsim_destroy(h);
        return fail(nullptr, rc, "initialisation failed");
    }
    *out = h;
    return QSIM_OK;
}

int qsim_create(int n, int ngpus, qsim_t **out)
{
    if (!out) return QSIM_EINVAL;
    *out = nullptr;
    if (ngpus < 1 || ngpus > 64 || (ngpus & (ngpus - 1)))
        return fail(nullptr, QSIM_EINVAL, "ngpus must be a power of two in [1, 64]");
    if (ngpus == 1) return create_common(n, 1, 0, -1, out);
    // several GPUs driven by this process: the rank-group path (one shard per
    // device, peer copies over NVLink), rank r on device r mod (device count)
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, QSIM_ENODEV, "no CUDA device (libqsim has no CPU path)");
    }
    std::vector<int> devs(ngpus);
    for (int r = 0; r < ngpus; ++r) devs[r] = r % ndev;
    return qsim_create_group(n, ngpus, devs.data(), out);
}

int qsim_create_dist(int n, int world, int rank, int device, const void *nccl_id, qsim_t **out)
{
    if (!out) return QSIM_EINVAL;
    if (rank < 0 || rank >= world) return fail(nullptr, QSIM_EINVAL, "rank outside [0, world)");
    int rc = create_common(n, world, rank, device, out);
    if (rc) return rc;
#ifndef QSIM_NO_NCCL
    if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof id);
        ncclResult_t r = ncclCommInitRank(&(*out)->comm, world, id, rank);
        if (r != ncclSuccess) {
            qsim_destroy(*out);
            *out = nullptr;
            return fail(nullptr, QSIM_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
    }
#else
    if (world > 1) {
        qsim_destroy(*out);
        *out = nullptr;
        return fail(nullptr, QSIM_ENCCL, "built without NCCL");
    }
#endif
    return QSIM_OK;
}

int qsim_create_group(int n, int world, const int *devices, qsim_t **out)
{
    if (!out) return QSIM_EINVAL;
    *out = nullptr;
    if (world < 1 || (world & (world - 1))) return fail(nullptr, QSIM_EINVAL, "world must be a power of two");
    qsim_t *g = new qsim_t();
    g->n = n;
    g->world = world;
    while ((1 << g->kglob) < world) ++g->kglob;
    g->nl = n - g->kglob;
    for (int q = 0; q < n && q < kMaxQubits; ++q) g->pos[q] = n - 1 - q;
    for (int r = 0; r < world; ++r) {
        qsim_t *m = nullptr;
        int rc = create_common(n, world, r, devices ? devices[r] : -1, &m);
        if (rc) {
            qsim_destroy(g);
            return rc;
        }
        m->grp = g;
        g->members.push_back(m);
    }
    // peer access between distinct member devices (NVLink peer copies)
    for (Handle *a : g->members)
        for (Handle *b : g->members)
            if (a->device != b->device) {
                cudaSetDevice(a->device);
                cudaDeviceEnablePeerAccess(b->device, 0);
                cudaGetLastError();
            }
    g->device = g->members[0]->device;
    g->stream = g->members[0]->stream;
    *out = g;
    return QSIM_OK;
}

int qsim_nccl_unique_id(void *out128)
{
#ifndef QSIM_NO_NCCL
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return QSIM_ENCCL;
    std::memcpy(out128, &id, sizeof id);
    return QSIM_OK;
#else
    (void)out128;
    return QSIM_ENCCL;
#endif
}

void qsim_destroy(qsim_t *h)
{
    if (!h) return;
    if (!h->members.empty()) {
        for (Handle *m : h->members) qsim_destroy(static_cast<qsim_t *>(m));
        h->members.clear();
        delete h;
        return;
    }
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
#ifndef QSIM_NO_NCCL
    if (h->comm) ncclCommDestroy(h->comm);
#endif
    for (size_t i = 0; i < h->peer_buf.size(); ++i)
        if ((int)(i / 2) != h->rank && h->peer_buf[i]) cudaIpcCloseMemHandle(h->peer_buf[i]);
    if (h->psi) cudaFree(h->psi);
    if (h->scratch) cudaFree(h->scratch);
    if (h->d_red) cudaFree(h->d_red);
    if (h->d_probs) cudaFree(h->d_probs);
    if (h->d_sum2) cudaFree(h->d_sum2);
    for (double2 *b : h->stage)
        if (b) cudaFree(b);
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    if (h->s_comm) {
        cudaStreamSynchronize(h->s_comm);
        cudaStreamDestroy(h->s_comm);
    }
    if (h->d_tabs) cudaFree(h->d_tabs);
    if (h->h_red) cudaFreeHost(h->h_red);
    for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

void *qsim_get_stream(qsim_t *h) { return h ? (void *)h->stream : nullptr; }

int qsim_set_fusion(qsim_t *h, int enable)
{
    QS_CHECK_HANDLE(h);
    const Ranks R = ranks_of(h);
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        if (int rc = flush_queue(m)) return lift(h, R, rc);
        m->fuse = enable ? 1 : 0;
    }
    h->fuse = enable ? 1 : 0;   // a group handle's own flag (read by qsim_qft) follows its members
    return QSIM_OK;
}

// profiling reports the first rank of a group
int qsim_profile(qsim_t *h, int enable)
{
    QS_CHECK_HANDLE(h);
    Handle *m = ranks_of(h)[0];
    if (int rc = flush_queue(m)) return rc;
    cudaStreamSynchronize(m->stream);
    m->prof.clear();
    m->ev_used = 0;
    m->pending = nullptr;
    m->prof_on = enable;
    return QSIM_OK;
}

const char *qsim_profile_json(qsim_t *h)
{
    if (!h) return "{}";
    Handle *m = ranks_of(h)[0];
    flush_queue(m);
    cudaStreamSynchronize(m->stream);
    struct Agg { double ms = 0; uint64_t bytes = 0, n = 0, fp64 = 0; };
    std::vector<std::pair<std::string, Agg>> agg;
    for (const auto &r : m->prof) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        size_t k = 0;
        while (k < agg.size() && agg[k].first != r.name) ++k;
        if (k == agg.size()) agg.push_back({r.name, Agg()});
        agg[k].second.ms += ms;
        agg[k].second.bytes += r.bytes;
        agg[k].second.n += 1;
        agg[k].second.fp64 += r.fp64;
    }
    std::string js = "{\"_launches\": [";
    char buf[256];
    for (size_t k = 0; k < m->prof.size() && k < 4096; ++k) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, m->prof[k].a, m->prof[k].b);
        std::snprintf(buf, sizeof buf, "%s[\"%s\", %.5f]", k ? ", " : "", m->prof[k].name, ms);
        js += buf;
    }
    js += "]";
    for (size_t k = 0; k < agg.size(); ++k) {
        std::snprintf(buf, sizeof buf, ", \"%s\": {\"launches\": %llu, \"ms\": %.6f, \"bytes\": %llu, \"fp64\": %llu}",
                      agg[k].first.c_str(), (unsigned long long)agg[k].second.n, agg[k].second.ms,
                      (unsigned long long)agg[k].second.bytes, (unsigned long long)agg[k].second.fp64);
        js += buf;
    }
    js += "}";
    h->prof_json = js;
    return h->prof_json.c_str();
}

int qsim_sync(qsim_t *h)
{
    QS_CHECK_HANDLE(h);
    const Ranks R = ranks_of(h);
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        if (int rc = flush_queue(m)) return lift(h, R, rc);
        if (int rc = check_cuda(m, cudaStreamSynchronize(m->stream), "qsim_sync")) return lift(h, R, rc);
#ifndef QSIM_NO_NCCL
        if (m->comm) {
            // an asynchronous NCCL failure (a peer died, a network error) surfaces here
            ncclResult_t ar = ncclSuccess;
            const ncclResult_t qr = ncclCommGetAsyncError(m->comm, &ar);
            if (qr != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
                m->poisoned = 1;
                return lift(h, R, fail(m, QSIM_ENCCL, std::string("NCCL asynchronous error: ") +
                                                           ncclGetErrorString(qr != ncclSuccess ? qr : ar)));
            }
        }
#endif
    }
    return QSIM_OK;
}

// ----------------------------------------------------------------- preparation
int qsim_set_basis(qsim_t *h, uint64_t idx)
{
    QS_CHECK_HANDLE(h);
    if (h->n < 64 && idx >> h->n) return fail(h, QSIM_ERANGE, "basis index >= 2^n");
    const Ranks R = ranks_of(h);
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        m->queue.clear();   // the state is overwritten
        for (int q = 0; q < m->n; ++q) m->pos[q] = m->n - 1 - q;
        launch_zero(m);
        if ((int)(idx >> m->nl) == m->rank) launch_set_one(m, idx & (m->local_dim() - 1));
        if (int rc = after_launch(m, "set_basis")) return lift(h, R, rc);
    }
    return QSIM_OK;
}

// sum |alpha|^2 over all ranks (fixed order)
static int global_norm(qsim_t *h, const Ranks &R, double *out)
{
    std::vector<std::vector<double>> parts(R.size(), std::vector<double>(1, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *m = R[i];
        cudaSetDevice(m->device);
        if (int rc = flush_queue(m)) return lift(h, R, rc);
        launch_norm(m, m->d_red);
        if (int rc = after_launch(m, "norm")) return lift(h, R, rc);
        if (int rc = check_cuda(m, cudaMemcpyAsync(m->h_red, m->d_red, sizeof(double), cudaMemcpyDeviceToHost, m->stream), "norm"))
            return lift(h, R, rc);
        if (int rc = check_cuda(m, cudaStreamSynchronize(m->stream), "norm")) return lift(h, R, rc);
        parts[i][0] = m->h_red[0];
    }
    return lift(h, R, dist_sum_host(R, parts, out, 1));
}

int qsim_init_gaussian(qsim_t *h, uint64_t seed)
{
    QS_CHECK_HANDLE(h);
    const Ranks R = ranks_of(h);
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        m->queue.clear();   // the state is overwritten
        for (int q = 0; q < m->n; ++q) m->pos[q] = m->n - 1 - q;
        launch_init_gaussian(m, seed);
    }
    double s = 0.0;
    if (int rc = global_norm(h, R, &s)) return rc;
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        launch_scale(m, 1.0 / std::sqrt(s));
        if (int rc = after_launch(m, "init_gaussian")) return lift(h, R, rc);
    }
    return QSIM_OK;
}

static int copy_state(qsim_t *h, uint64_t off, uint64_t cnt, qsim_c128 *host, bool to_dev)
{
    QS_CHECK_HANDLE(h);
    const uint64_t dim = (uint64_t)1 << h->n;
    if (off > dim || cnt > dim - off) return fail(h, QSIM_ERANGE, "state slice outside [0, 2^n)");
    const Ranks R = ranks_of(h);
    if (int rc = dist_canonicalize(R)) return lift(h, R, rc);
    // an in-process group owns every slice; a process rank only its own
    if (R.size() == 1 && cnt) {
        Handle *m = R[0];
        const uint64_t lo = (uint64_t)m->rank << m->nl, hi = lo + m->local_dim();
        if (off < lo || off + cnt > hi) return fail(h, QSIM_ERANGE, "slice not owned by this rank");
    }
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        const uint64_t lo = (uint64_t)m->rank << m->nl, hi = lo + m->local_dim();
        const uint64_t a = std::max(off, lo), b = std::min(off + cnt, hi);
        if (a >= b) continue;
        cudaError_t e;
        if (to_dev)
            e = cudaMemcpyAsync(m->psi + (a - lo), host + (a - off), (b - a) * sizeof(double2), cudaMemcpyHostToDevice, m->stream);
        else
            e = cudaMemcpyAsync(host + (a - off), m->psi + (a - lo), (b - a) * sizeof(double2), cudaMemcpyDeviceToHost, m->stream);
        if (e != cudaSuccess) return lift(h, R, check_cuda(m, e, "state copy"));
        if (int rc = check_cuda(m, cudaStreamSynchronize(m->stream), "state copy")) return lift(h, R, rc);
    }
    return QSIM_OK;
}

int qsim_set_state(qsim_t *h, uint64_t off, uint64_t cnt, const qsim_c128 *host)
{
    return copy_state(h, off, cnt, const_cast<qsim_c128 *>(host), true);
}

int qsim_get_state(qsim_t *h, uint64_t off, uint64_t cnt, qsim_c128 *host)
{
    return copy_state(h, off, cnt, host, false);
}

// ----------------------------------------------------------------- gates
int qsim_apply_1q(qsim_t *h, int q, const qsim_c128 U[4])
{
    QS_CHECK_HANDLE(h);
    if (int rc = check_qubit(h, q)) return rc;
    double2 M[4];
    for (int k = 0; k < 4; ++k) M[k] = make_double2(U[k].re, U[k].im);
    if (int rc = check_unitary(h, M)) return rc;
    const Ranks R = ranks_of(h);
    return lift(h, R, apply_gate(R, 0, 0, q, M));
}

int qsim_set_strict(qsim_t *h, int enable)
{
    QS_CHECK_HANDLE(h);
    h->strict = enable ? 1 : 0;
    return QSIM_OK;
}

int qsim_apply_ctrl(qsim_t *h, uint64_t cmask, uint64_t cvals, int q, const qsim_c128 U[4])
{
    QS_CHECK_HANDLE(h);
    if (int rc = check_qubit(h, q)) return rc;
    if (int rc = check_ctrl(h, cmask, cvals, q)) return rc;
    double2 M[4];
    for (int k = 0; k < 4; ++k) M[k] = make_double2(U[k].re, U[k].im);
    if (int rc = check_unitary(h, M)) return rc;
    const Ranks R = ranks_of(h);
    return lift(h, R, apply_gate(R, cmask, cvals, q, M));
}

// A table of 4 * B matrices in the member's arena (batch.cu); the member's
// queue is flushed first when the producers' half of the arena is full
// (flushing consumes every queued table, stream-ordered).  The other half
// takes the planner's merged products (plan_ops.cu try_merge_tab).
static double2 *batch_table(Handle *m, uint64_t B, int &rc)
{
    rc = QSIM_OK;
    const size_t need = 4 * B;
    if (m->tabs_used + need > m->tabs_cap / 2) {
        if ((rc = flush_queue(m))) return nullptr;
        m->tabs_used = 0;
        if (need > m->tabs_cap / 2) {
            if (m->d_tabs) {
                cudaStreamSynchronize(m->stream);
                cudaFree(m->d_tabs);
            }
            m->d_tabs = nullptr;
            m->tabs_cap = 0;
            // ~1000 tables per half at 2^10 trajectories (128 MiB), <= 256 MiB
            const size_t cap = std::max<size_t>(std::min<size_t>(need * 2048, (size_t)1 << 24), 2 * need);
            if (cudaMalloc(&m->d_tabs, cap * sizeof(double2)) != cudaSuccess) {
                cudaGetLastError();
                rc = fail(m, QSIM_ENOMEM, "batch matrix tables");
                return nullptr;
            }
            m->tabs_cap = cap;
        }
    }
    double2 *p = m->d_tabs + m->tabs_used;
    m->tabs_used += need;
    return p;
}

int qsim_apply_angles(qsim_t *h, int kind, const double *ang, uint64_t cmask, uint64_t cvals, int q)
{
    QS_CHECK_HANDLE(h);
    if (kind < 0 || kind > 2 || !ang) return fail(h, QSIM_EINVAL, "unknown angle-form gate kind");
    if (int rc = check_qubit(h, q)) return rc;
    if (int rc = check_ctrl(h, cmask, cvals, q)) return rc;
    if (h->batch_b > 0 && h->sigma > 0.0) {
        // batched trajectories: one perturbed matrix per trajectory, drawn on
        // the device from seed + t (R33)
        if (q < h->batch_b || (cmask & ((1ull << h->batch_b) - 1)))
            return fail(h, QSIM_EINVAL, "gate on a trajectory-index qubit of a batched handle");
        const Ranks R = ranks_of(h);
        const uint64_t B = 1ull << h->batch_b;
        std::vector<const double2 *> tabs;
        for (Handle *m : R) {
            int rc;
            double2 *t = batch_table(m, B, rc);
            if (!t) return lift(h, R, rc);
            launch_batch_mats(m, kind, ang, h->sigma, h->noise_seed, h->gcount, B, t);
            if ((rc = after_launch(m, "batch matrices"))) return lift(h, R, rc);
            tabs.push_back(t);
        }
        h->gcount++;
        const double2 X[4] = {make_double2(0, 0), make_double2(1, 0), make_double2(1, 0), make_double2(0, 0)};
        return lift(h, R, apply_gate(R, cmask, cvals, q, X, &tabs));
    }
    double2 U[4];
    angle_matrix(h, kind, ang, h->gcount, U);
    h->gcount++;
    const Ranks R = ranks_of(h);
    return lift(h, R, apply_gate(R, cmask, cvals, q, U));
}

int qsim_apply_gates(qsim_t *h, const qsim_gate_t *gates, int count, int *done)
{
    QS_CHECK_HANDLE(h);
    if (done) *done = 0;
    if (count < 0 || (count > 0 && !gates)) return fail(h, QSIM_EINVAL, "gate list");
    for (int i = 0; i < count; ++i) {
        const qsim_gate_t &g = gates[i];
        int rc;
        if (g.type == QSIM_GT_MATRIX)
            rc = g.ctrl_mask ? qsim_apply_ctrl(h, g.ctrl_mask, g.ctrl_vals, g.q, g.U) : qsim_apply_1q(h, g.q, g.U);
        else if (g.type == QSIM_GT_ANGLES)
            rc = qsim_apply_angles(h, g.akind, g.ang, g.ctrl_mask, g.ctrl_vals, g.q);
        else
            rc = fail(h, QSIM_EINVAL, "unknown gate type in the list");
        if (rc) return rc;
        if (done) *done = i + 1;
    }
    return QSIM_OK;
}

int qsim_set_gate_noise(qsim_t *h, uint64_t seed, double sigma)
{
    QS_CHECK_HANDLE(h);
    if (!(sigma >= 0.0)) return fail(h, QSIM_EINVAL, "sigma must be >= 0");
    h->noise_seed = seed;
    h->sigma = sigma;
    return QSIM_OK;
}

int qsim_get_gate_counter(const qsim_t *h, uint64_t *g)
{
    if (!h || !g) return QSIM_EINVAL;
    *g = h->gcount;
    return QSIM_OK;
}

int qsim_set_gate_counter(qsim_t *h, uint64_t g)
{
    QS_CHECK_HANDLE(h);
    h->gcount = g;
    return QSIM_OK;
}

int qsim_swap(qsim_t *h, int q1, int q2)
{
    QS_CHECK_HANDLE(h);
    if (int rc = check_qubit(h, q1)) return rc;
    if (int rc = check_qubit(h, q2)) return rc;
    // a SWAP is a relabelling of the logical -> physical map (no data moves;
    // queued gates already carry physical positions)
    for (Handle *m : ranks_of(h)) std::swap(m->pos[q1], m->pos[q2]);
    return QSIM_OK;
}

static int fused_qft_gen(qsim_t *h, const Ranks &R, int lo, int m, int band, int inverse, bool honly);

int qsim_hadamard(qsim_t *h, int lo, int m)
{
    QS_CHECK_HANDLE(h);
    if (lo < 0 || m < 0 || lo + m > h->n) return fail(h, QSIM_ERANGE, "range outside [0, n)");
    if (m == 0) return QSIM_OK;
    const Ranks R = ranks_of(h);
    if (h->nl >= 9 && (m <= h->nl || h->nl >= 12)) return lift(h, R, fused_range(R, lo, m, 0, 0));
    const double r = M_SQRT1_2;
    double2 H[4] = {make_double2(r, 0), make_double2(r, 0), make_double2(r, 0), make_double2(-r, 0)};
    for (int q = lo; q < lo + m; ++q)
        if (int rc = apply_gate(R, 0, 0, q, H)) return lift(h, R, rc);
    return QSIM_OK;
}

// The QFT circuit of PAPER.md:442-469 gate by gate through the gate queue
// (fused into tile passes at the next flush): H(lo+j), R_{k-j} controlled by
// lo+k on lo+j for k - j <= band, closing swaps as relabels.  With gate noise
// every H / R_d is an angle-form gate (R14/R15); count = advance the gate
// counter per applied gate.
static int qft_gates(qsim_t *h, const Ranks &R, int lo, int m, int band, int inverse, bool count)
{
    const double sgn = inverse ? -1.0 : 1.0;
    const double r = M_SQRT1_2;
    const double2 H[4] = {make_double2(r, 0), make_double2(r, 0), make_double2(r, 0), make_double2(-r, 0)};
    const bool noisy = count && h->sigma > 0.0;
    for (int j = 0; j < m; ++j) {
        int rc;
        if (noisy) {
            const double ang[2] = {M_PI / 4.0, M_PI};
            rc = qsim_apply_angles(h, QSIM_GATE_RP, ang, 0, 0, lo + j);
        } else {
            rc = lift(h, R, apply_gate(R, 0, 0, lo + j, H));
            if (count) h->gcount++;
        }
        if (rc) return rc;
        for (int k = j + 1; k < m; ++k) {
            if (k - j > band) continue;
            const double phi = sgn * M_PI / std::ldexp(1.0, k - j);
            const uint64_t cm = 1ull << (lo + k);
            if (noisy) {
                rc = qsim_apply_angles(h, QSIM_GATE_P1, &phi, cm, cm, lo + j);
            } else {
                double2 Rd[4] = {make_double2(1, 0), make_double2(0, 0), make_double2(0, 0),
                                 make_double2(std::cos(phi), std::sin(phi))};
                rc = lift(h, R, apply_gate(R, cm, cm, lo + j, Rd));
                if (count) h->gcount++;
            }
            if (rc) return rc;
        }
    }
    for (Handle *mm : R)
        for (int j = 0; j < m / 2; ++j) std::swap(mm->pos[lo + j], mm->pos[lo + m - 1 - j]);
    return QSIM_OK;
}

// qft_gates(h, R, lo, m, band, inverse, count = true) as fused passes
// (k_qft_gen): the matrices and angles the gate-by-gate path would apply --
// the same Philox draws, in the same gate-counter order -- handed to the
// generalised kernel.  Returns 1 (nothing done) when the register does not
// fit the pass geometry; the caller then runs qft_gates.
static int fused_qft_gen(qsim_t *h, const Ranks &R, int lo, int m, int band, int inverse, bool honly)
{
    static const bool off = getenv("QSIM_NO_QFT_GEN") != nullptr;
    if (off || h->world != 1 || R.size() != 1 || h->batch_b > 0 || !h->fuse || h->nl < 9 || m > h->nl || m < 4 ||
        m > kGenEarly)
        return 1;
    // geometry first: a dry run changes nothing but the canonicalisation / flush
    // fused_range does anyway (its closing-swap relabel is skipped when dry)
    GenCircuit gc;
    gc.m = m;
    bool even = false;
    int rc = fused_range(R, lo, m, honly ? 0 : 1, inverse, &gc, true, false);
    if (rc == kGenInfeasible) {
        even = true;
        rc = fused_range(R, lo, m, honly ? 0 : 1, inverse, &gc, true, true);
    }
    if (rc == kGenInfeasible) return 1;
    if (rc) return lift(h, R, rc);
    const double sgn = inverse ? -1.0 : 1.0;
    const double r = M_SQRT1_2;
    const bool noisy = h->sigma > 0.0;
    gc.Hr.assign(4 * m, 0.0);
    gc.hph.assign(m, 0.0);
    gc.phi.assign((size_t)m * m, 0.0);
    gc.e.assign((size_t)m * m, make_double2(1, 0));
    uint64_t g = h->gcount;
    for (int j = 0; j < m; ++j) {
        // H = RP(pi/4, pi) = U_R(a0) U_P1(a1) = [[c, -s], [s, c]] diag(1, e^{i a1}) (R14)
        double Hr[4] = {r, r, r, -r}, ph = 0.0;
        if (noisy) {
            const double ang[2] = {M_PI / 4.0, M_PI};
            double a[4];
            noisy_angles(h, QSIM_GATE_RP, ang, g, a);
            const double c = std::cos(a[0]), s = std::sin(a[0]);
            Hr[0] = c; Hr[1] = -s; Hr[2] = s; Hr[3] = c;
            ph = a[1];
        }
        g++;
        for (int k = 0; k < 4; ++k) gc.Hr[4 * j + k] = Hr[k];
        gc.hph[j] = ph;
        for (int k = j + 1; k < m; ++k) {
            if (k - j > band) continue;
            double phi = sgn * M_PI / std::ldexp(1.0, k - j);
            if (noisy) {
                double a[4];
                noisy_angles(h, QSIM_GATE_P1, &phi, g, a);
                phi = a[0];
            }
            gc.e[(size_t)j * m + k] = make_double2(std::cos(phi), std::sin(phi));
            gc.phi[(size_t)j * m + k] = phi;
            g++;
        }
    }
    if ((rc = fused_range(R, lo, m, honly ? 0 : 1, inverse, &gc, false, even))) return lift(h, R, rc);
    h->gcount = g;
    return QSIM_OK;
}

int qsim_hadamard_angles(qsim_t *h, int lo, int m)
{
    QS_CHECK_HANDLE(h);
    if (lo < 0 || m < 0 || lo + m > h->n) return fail(h, QSIM_ERANGE, "range outside [0, n)");
    if (m == 0) return QSIM_OK;
    const Ranks R = ranks_of(h);
    if (h->sigma > 0.0) {
        // the generalised QFT passes with no R_d (band 0) in Hadamard mode
        // (passes in place, no block moves): H(lo+j) drawn at counter g0 + j
        // as in the gate-by-gate loop
        const int rc = fused_qft_gen(h, R, lo, m, 0, 0, true);
        if (rc != 1) return rc;
    }
    const double ang[2] = {M_PI / 4.0, M_PI};
    for (int q = lo; q < lo + m; ++q)
        if (int rc = qsim_apply_angles(h, QSIM_GATE_RP, ang, 0, 0, q)) return rc;
    return QSIM_OK;
}

int qsim_qft(qsim_t *h, int lo, int m, int inverse)
{
    QS_CHECK_HANDLE(h);
    if (lo < 0 || m < 0 || lo + m > h->n) return fail(h, QSIM_ERANGE, "range outside [0, n)");
    if (m == 0) return QSIM_OK;
    const Ranks R = ranks_of(h);
    if (h->sigma == 0.0 && h->fuse && h->nl >= 9 && (m <= h->nl || h->nl >= 12)) {
        // noiseless: fused passes (constant gates, R25)
        h->gcount += (uint64_t)m + (uint64_t)m * (m - 1) / 2;
        return lift(h, R, fused_range(R, lo, m, 1, inverse));
    }
    if (h->sigma > 0.0) {
        // operational error: the perturbed gates as fused passes when the geometry allows
        const int rc = fused_qft_gen(h, R, lo, m, m, inverse, false);
        if (rc != 1) return rc;
    }
    // noisy, or fusion off (the paper's one sweep per gate)
    return qft_gates(h, R, lo, m, m, inverse, true);
}

// QFT of `count` host-resident states, pipelined: state i+1 is copied in
// (its own stream) while state i is transformed and state i-1 copied out
// (a third stream).  Four shard buffers (psi, scratch, two stages) rotate;
// cross-stream order comes from events recorded on the streams that last
// used each buffer.  Every transform is qsim_qft's own fused pass plan.
int qsim_qft_host_stream(qsim_t *h, int lo, int m, int inverse, const qsim_c128 *in, uint64_t in_stride,
                         qsim_c128 *out, uint64_t out_stride, int count)
{
    QS_CHECK_HANDLE(h);
    if (lo < 0 || m < 1 || lo + m > h->n) return fail(h, QSIM_ERANGE, "range outside [0, n)");
    if (count < 0 || (count > 0 && (!in || !out))) return fail(h, QSIM_EINVAL, "host buffers / count");
    if (h->world != 1 || !h->members.empty() || h->batch_b)
        return fail(h, QSIM_EINVAL, "qsim_qft_host_stream runs on a single-GPU handle");
    if (h->sigma != 0.0) return fail(h, QSIM_EINVAL, "qsim_qft_host_stream: noiseless transforms only");
    if (count == 0) return QSIM_OK;
    const Ranks R = ranks_of(h);
    cudaSetDevice(h->device);
    if (int rc = flush_queue(h)) return rc;
    if (int rc = ensure_scratch(h)) return rc;
    for (double2 *&b : h->stage)
        if (!b && check_cuda(h, cudaMalloc(&b, sizeof(double2) * h->local_dim()), "stream stage buffer"))
            return QSIM_ENOMEM;
    if (!h->s_h2d && check_cuda(h, cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking), "copy stream"))
        return QSIM_ECUDA;
    if (!h->s_d2h && check_cuda(h, cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking), "copy stream"))
        return QSIM_ECUDA;
    for (int q = 0; q < h->n; ++q) h->pos[q] = h->n - 1 - q;   // each input is given in the canonical layout
    const size_t bytes = sizeof(double2) * h->local_dim();
    double2 *buf[4] = {h->psi, h->scratch, h->stage[0], h->stage[1]};
    cudaEvent_t done[4];   // last use of each buffer (any stream)
    for (auto &e : done) {
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        cudaEventRecord(e, h->stream);
    }
    auto idx_of = [&](const double2 *p) {
        for (int b = 0; b < 4; ++b)
            if (buf[b] == p) return b;
        return -1;
    };
    int busy_out = -1, busy_out2 = -1;   // buffers still being copied out (states i-1, i-2)
    int in_next = 2;                     // buffer the next input lands in
    int rc = QSIM_OK;
    // first input
    cudaStreamWaitEvent(h->s_h2d, done[in_next], 0);
    rc = check_cuda(h, cudaMemcpyAsync(buf[in_next], in, bytes, cudaMemcpyHostToDevice, h->s_h2d), "stream H2D");
    for (int i = 0; i < count && !rc; ++i) {
        const int cur = in_next;
        cudaEvent_t landed;
        cudaEventCreateWithFlags(&landed, cudaEventDisableTiming);
        cudaEventRecord(landed, h->s_h2d);
        cudaStreamWaitEvent(h->stream, landed, 0);
        cudaEventDestroy(landed);
        // the compute scratch: a buffer that is neither the input nor being copied out
        int sc = -1;
        for (int b = 0; b < 4 && sc < 0; ++b)
            if (b != cur && b != busy_out && b != busy_out2) sc = b;
        cudaStreamWaitEvent(h->stream, done[sc], 0);
        h->psi = buf[cur];
        h->scratch = buf[sc];
        rc = fused_range(R, lo, m, 1, inverse);
        if (rc) break;
        h->gcount += (uint64_t)m + (uint64_t)m * (m - 1) / 2;
        const int res = idx_of(h->psi), other = idx_of(h->scratch);
        cudaEventRecord(done[other], h->stream);
        cudaEventRecord(done[res], h->stream);
        // the next input: a buffer not holding this result, not being copied out
        if (i + 1 < count) {
            in_next = -1;
            for (int b = 0; b < 4 && in_next < 0; ++b)
                if (b != res && b != busy_out && b != other) in_next = b;
            if (in_next < 0) in_next = other;
            cudaStreamWaitEvent(h->s_h2d, done[in_next], 0);
            rc = check_cuda(h, cudaMemcpyAsync(buf[in_next], in + (size_t)(i + 1) * in_stride, bytes, cudaMemcpyHostToDevice,
                                               h->s_h2d), "stream H2D");
            if (rc) break;
        }
        // copy the result out once the transform is done
        cudaStreamWaitEvent(h->s_d2h, done[res], 0);
        rc = check_cuda(h, cudaMemcpyAsync(out + (size_t)i * out_stride, buf[res], bytes, cudaMemcpyDeviceToHost, h->s_d2h),
                        "stream D2H");
        cudaEventRecord(done[res], h->s_d2h);
        busy_out2 = busy_out;
        busy_out = res;
    }
    if (!rc) rc = check_cuda(h, cudaStreamSynchronize(h->s_h2d), "stream H2D");
    if (!rc) rc = check_cuda(h, cudaStreamSynchronize(h->stream), "stream compute");
    if (!rc) rc = check_cuda(h, cudaStreamSynchronize(h->s_d2h), "stream D2H");
    for (auto &e : done) cudaEventDestroy(e);
    // the handle keeps the last result as its state; the other buffers as scratch / stages
    const int res = idx_of(h->psi);
    int k = 0;
    for (int b = 0; b < 4; ++b) {
        if (b == res) continue;
        if (k == 0) h->scratch = buf[b];
        else h->stage[k - 1] = buf[b];
        ++k;
    }
    return rc;
}

int qsim_fft(qsim_t *h, int lo, int m, int inverse)
{
    QS_CHECK_HANDLE(h);
    if (lo < 0 || m < 0 || lo + m > h->n) return fail(h, QSIM_ERANGE, "range outside [0, n)");
    if (m == 0) return QSIM_OK;
    const Ranks R = ranks_of(h);
    if (h->nl >= 9 && (m <= h->nl || h->nl >= 12)) return lift(h, R, fused_range(R, lo, m, 1, inverse));
    return qft_gates(h, R, lo, m, m, inverse, false);   // tiny registers: constant gates, not counted
}

int qsim_aqft(qsim_t *h, int lo, int m, int b, int inverse)
{
    QS_CHECK_HANDLE(h);
    if (lo < 0 || m < 0 || lo + m > h->n || b < 0) return fail(h, QSIM_ERANGE, "range outside [0, n) or b < 0");
    if (m == 0) return QSIM_OK;
    if (b >= m - 1) return qsim_qft(h, lo, m, inverse);
    const Ranks R = ranks_of(h);
    const int rc = fused_qft_gen(h, R, lo, m, b, inverse, false);
    if (rc != 1) return rc;
    return qft_gates(h, R, lo, m, b, inverse, true);
}

int qsim_phase_flip(qsim_t *h, uint64_t idx)
{
    QS_CHECK_HANDLE(h);
    if (h->n < 64 && idx >> h->n) return fail(h, QSIM_ERANGE, "index >= 2^n");
    const Ranks R = ranks_of(h);
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        if (int rc = flush_queue(m)) return lift(h, R, rc);
        // physical location of logical index idx
        uint64_t phys = 0;
        for (int q = 0; q < m->n; ++q) phys |= ((idx >> (m->n - 1 - q)) & 1) << m->pos[q];
        if ((int)(phys >> m->nl) != m->rank) continue;
        const uint64_t mask = m->local_dim() - 1;
        launch_phase_mask(m, mask, phys & mask, make_double2(-1.0, 0.0));
        if (int rc = after_launch(m, "phase_flip")) return lift(h, R, rc);
    }
    return QSIM_OK;
}

// D = 2|s><s| - I on the whole register in the mean form alpha <- 2 mean -
// alpha: one read-only pass for the sum (fixed tree per shard, shards summed
// on the host in rank order), one update pass.  The sum and the update are
// layout-independent, so no exchange or canonicalisation is needed.
static int diffusion_mean(qsim_t *h, const Ranks &R)
{
    std::vector<std::vector<double>> parts(R.size(), std::vector<double>(2, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *m = R[i];
        cudaSetDevice(m->device);
        if (int rc = flush_queue(m)) return rc;
        if (!m->d_sum2 && check_cuda(m, cudaMalloc(&m->d_sum2, 2 * sizeof(double)), "diffusion buffer")) return QSIM_ECUDA;
        ensure_hred(m, 2);
        launch_amp_sum(m, m->d_sum2);
        if (int rc = after_launch(m, "diffusion sum")) return rc;
        if (int rc = check_cuda(m, cudaMemcpyAsync(m->h_red, m->d_sum2, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                                   m->stream), "diffusion"))
            return rc;
    }
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *m = R[i];
        cudaSetDevice(m->device);
        if (int rc = check_cuda(m, cudaStreamSynchronize(m->stream), "diffusion")) return rc;
        parts[i][0] = m->h_red[0];
        parts[i][1] = m->h_red[1];
    }
    double S[2];
    if (int rc = dist_sum_host(R, parts, S, 2)) return rc;
    const double inv = std::ldexp(1.0, -h->n);
    const double2 c = make_double2(2.0 * S[0] * inv, 2.0 * S[1] * inv);
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        launch_reflect(m, c);
        if (int rc = after_launch(m, "diffusion")) return rc;
    }
    return QSIM_OK;
}

int qsim_diffusion(qsim_t *h, int lo, int m)
{
    QS_CHECK_HANDLE(h);
    if (lo < 0 || m < 1 || lo + m > h->n) return fail(h, QSIM_ERANGE, "range outside [0, n) or m < 1");
    const Ranks R = ranks_of(h);
    if (lo == 0 && m == h->n && !h->batch_b) return lift(h, R, diffusion_mean(h, R));
    // a sub-register: the paper's literal -H_m V_{f0} H_m, with
    // -V_{f0} = 2|0><0| - I as two diagonal gates: a global -1 and a flip of
    // the range value 0 (controls on lo..lo+m-2 at 0, target lo+m-1)
    if (int rc = qsim_hadamard(h, lo, m)) return rc;
    const double2 minus[4] = {make_double2(-1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(-1, 0)};
    const double2 flip0[4] = {make_double2(-1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0)};
    uint64_t cm = 0;
    for (int q = lo; q < lo + m - 1; ++q) cm |= 1ull << q;
    if (int rc = lift(h, R, apply_gate(R, 0, 0, lo + m - 1, minus))) return rc;
    if (int rc = lift(h, R, apply_gate(R, cm, 0, lo + m - 1, flip0))) return rc;
    return qsim_hadamard(h, lo, m);
}

int qsim_grover(qsim_t *h, uint64_t mark, int iters, double *trace)
{
    QS_CHECK_HANDLE(h);
    if (h->n < 64 && mark >> h->n) return fail(h, QSIM_ERANGE, "mark >= 2^n");
    if (iters < 0) return fail(h, QSIM_EINVAL, "iters < 0");
    if (h->batch_b) return fail(h, QSIM_EINVAL, "qsim_grover on a batched handle (use gates)");
    const Ranks R = ranks_of(h);
    if (h->world > 1) {
        // sharded: per iteration the phase flip on the owner rank, the mean-form
        // diffusion with the fixed-order cross-rank sum, and the trace read
        for (int t = 0; t < iters; ++t) {
            if (int rc = qsim_phase_flip(h, mark)) return rc;
            if (int rc = lift(h, R, diffusion_mean(h, R))) return rc;
            if (trace)
                if (int rc = qsim_prob_index(h, mark, trace + t)) return rc;
        }
        return QSIM_OK;
    }
    if (int rc = dist_canonicalize(R)) return rc;
    double *d_trace = nullptr;
    if (trace && iters > 0) {
        if (cudaMalloc(&d_trace, sizeof(double) * iters) != cudaSuccess) {
            cudaGetLastError();
            return fail(h, QSIM_ENOMEM, "cannot allocate the trace buffer");
        }
    }
    launch_grover(h, mark, 0, iters, d_trace);
    int rc = after_launch(h, "grover");
    if (!rc && d_trace) {
        rc = check_cuda(h, cudaMemcpyAsync(trace, d_trace, sizeof(double) * iters, cudaMemcpyDeviceToHost, h->stream),
                        "grover trace");
        if (!rc) rc = check_cuda(h, cudaStreamSynchronize(h->stream), "grover trace");
    }
    if (d_trace) cudaFree(d_trace);
    return rc;
}

// ----------------------------------------------------------------- permutations
static uint64_t gcd64(uint64_t a, uint64_t b)
{
    while (b) { uint64_t t = a % b; a = b; b = t; }
    return a;
}

int qsim_apply_perm(qsim_t *h, const qsim_perm_t *f)
{
    QS_CHECK_HANDLE(h);
    if (!f) return fail(h, QSIM_EINVAL, "null permutation");
    if (f->kind < 0 || f->kind > 2) return fail(h, QSIM_EINVAL, "unknown permutation kind");
    if (f->m < 1 || f->lo < 0 || f->lo + f->m > h->n) return fail(h, QSIM_ERANGE, "target register outside [0, n)");
    uint64_t treg = ((f->m >= 64) ? ~0ull : ((1ull << f->m) - 1)) << f->lo;
    if (f->ctrl_mask & treg) return fail(h, QSIM_EINVAL, "control overlaps the target register");
    if (f->ctrl_vals & ~f->ctrl_mask) return fail(h, QSIM_EINVAL, "ctrl_vals outside ctrl_mask");
    if (h->n < 64 && (f->ctrl_mask >> h->n)) return fail(h, QSIM_ERANGE, "control mask has qubits >= n");
    if (f->kind == QSIM_PERM_TABLE) {
        if (f->m > 24 || !f->table) return fail(h, QSIM_EINVAL, "TABLE needs m <= 24 and a table");
        const uint64_t len = 1ull << f->m;
        std::vector<char> seen(len, 0);
        for (uint64_t v = 0; v < len; ++v) {
            if (f->table[v] >= len || seen[f->table[v]]) return fail(h, QSIM_ENOTBIJ, "table is not a bijection");
            seen[f->table[v]] = 1;
        }
    } else {
        const uint64_t N = f->modulus;
        if (N < 2 || N >= (1ull << 32) || (f->m < 64 && N > (1ull << f->m)))
            return fail(h, QSIM_EINVAL, "modulus must be in [2, min(2^m, 2^32))");
        const uint64_t c = f->kind == QSIM_PERM_MODMUL ? f->mult : f->base;
        if (gcd64(c % N, N) != 1) return fail(h, QSIM_ENOTBIJ, "multiplier not coprime to the modulus");
        if (f->kind == QSIM_PERM_MODEXP) {
            if (f->em < 1 || f->em > 40 || f->elo < 0 || f->elo + f->em > h->n)
                return fail(h, QSIM_ERANGE, "exponent register outside [0, n)");
            uint64_t ereg = ((1ull << f->em) - 1) << f->elo;
            if (ereg & (treg | f->ctrl_mask)) return fail(h, QSIM_EINVAL, "exponent register overlaps");
        }
    }
    const Ranks R = ranks_of(h);
    if (int rc = flush_all(R)) return lift(h, R, rc);
    // the work register must be local (exponent / control qubits may be rank bits)
    std::vector<int> need;
    for (int q = f->lo; q < f->lo + f->m; ++q) need.push_back(q);
    if (int rc = dist_make_local(R, need)) return lift(h, R, rc);
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        PermDesc d;
        std::memset(&d, 0, sizeof d);
        d.kind = f->kind;
        d.wm = f->m;
        d.mult = f->mult;
        d.base = f->base;
        d.modulus = f->modulus;
        // work value bit b (LSB) <-> logical qubit lo+m-1-b
        for (int b = 0; b < f->m; ++b) d.wpos[b] = m->pos[f->lo + f->m - 1 - b];
        if (f->kind == QSIM_PERM_MODEXP) {
            d.em = f->em;
            for (int b = 0; b < f->em; ++b) {
                const int p = m->pos[f->elo + f->em - 1 - b];
                d.epos[b] = p < m->nl ? p : -1 - (p - m->nl);
            }
        }
        uint64_t lm, lv;
        if (!local_controls(m, f->ctrl_mask, f->ctrl_vals, lm, lv)) continue;
        d.cmask = lm;
        d.cval = lv;
        d.rank_bits = (uint64_t)m->rank;
        uint32_t *d_table = nullptr;
        if (f->kind == QSIM_PERM_TABLE) {
            const uint64_t len = 1ull << f->m;
            if (cudaMalloc(&d_table, sizeof(uint32_t) * len) != cudaSuccess) {
                cudaGetLastError();
                return fail(h, QSIM_ENOMEM, "cannot allocate the permutation table");
            }
            cudaMemcpyAsync(d_table, f->table, sizeof(uint32_t) * len, cudaMemcpyHostToDevice, m->stream);
            d.d_table = d_table;
        }
        int rc = launch_perm(m, d);
        if (!rc) rc = after_launch(m, "permutation");
        if (d_table) { cudaStreamSynchronize(m->stream); cudaFree(d_table); }
        if (rc) return lift(h, R, rc);
    }
    return QSIM_OK;
}

// ----------------------------------------------------------------- decoherence
int qsim_inject_errors(qsim_t *h, uint64_t seed, const qsim_noise_t *model, qsim_event_t *ev, int cap,
                       int *nev)
{
    QS_CHECK_HANDLE(h);
    if (!model) return fail(h, QSIM_EINVAL, "null noise model");
    if (!(model->p >= 0.0 && model->p <= 1.0)) return fail(h, QSIM_EINVAL, "p must be in [0, 1]");
    const Ranks R = ranks_of(h);
    int count = 0;
    if (h->batch_b > 0) {
        // batched trajectories (R33): trajectory t draws from seed + t; the
        // Paulis of one qubit become one per-trajectory table gate (identity
        // where no event); events in qubit order, then trajectory order
        const int b = h->batch_b;
        const uint64_t B = 1ull << b;
        if (model->qubit_mask & ((1ull << b) - 1))
            return fail(h, QSIM_EINVAL, "Pauli injection on trajectory-index qubits");
        std::vector<double2> tab(4 * B);
        const double p = model->p;
        for (int q = b; q < h->n; ++q) {
            if (!((model->qubit_mask >> q) & 1)) continue;
            bool any = false;
            for (uint64_t t = 0; t < B; ++t) {
                // the register's own qubit index: trajectory t is the single-register circuit (R33)
                const u64x2 d = draw(seed + t, QSIM_TAG_PAULI, model->epoch, (uint32_t)(q - b));
                const double u = u01(d.a);
                const int which = u < p / 3.0 ? 1 : u < 2.0 * p / 3.0 ? 2 : u < p ? 3 : 0;
                double2 *P = &tab[4 * t];
                if (which == 1) { P[0] = make_double2(0, 0); P[1] = make_double2(1, 0); P[2] = make_double2(1, 0); P[3] = make_double2(0, 0); }
                else if (which == 2) { P[0] = make_double2(0, 0); P[1] = make_double2(0, -1); P[2] = make_double2(0, 1); P[3] = make_double2(0, 0); }
                else if (which == 3) { P[0] = make_double2(1, 0); P[1] = make_double2(0, 0); P[2] = make_double2(0, 0); P[3] = make_double2(-1, 0); }
                else { P[0] = make_double2(1, 0); P[1] = make_double2(0, 0); P[2] = make_double2(0, 0); P[3] = make_double2(1, 0); }
                if (!which) continue;
                any = true;
                if (ev && count < cap) {
                    ev[count].epoch = model->epoch;
                    ev[count].qubit = q;
                    ev[count].pauli = which;
                    ev[count].traj = t;
                }
                ++count;
            }
            if (!any) continue;
            std::vector<const double2 *> tabs;
            for (Handle *m : R) {
                cudaSetDevice(m->device);
                int rc;
                double2 *dt = batch_table(m, B, rc);
                if (!dt) return lift(h, R, rc);
                // pageable source: consumed before the call returns
                if ((rc = check_cuda(m, cudaMemcpyAsync(dt, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice, m->stream), "pauli table")))
                    return lift(h, R, rc);
                tabs.push_back(dt);
            }
            const double2 X[4] = {make_double2(0, 0), make_double2(1, 0), make_double2(1, 0), make_double2(0, 0)};
            if (int rc = apply_gate(R, 0, 0, q, X, &tabs)) return lift(h, R, rc);
        }
        if (nev) *nev = count;
        if (ev && count > cap) return fail(h, QSIM_ERANGE, "event buffer too small");
        return QSIM_OK;
    }
    for (int q = 0; q < h->n; ++q) {
        if (!((model->qubit_mask >> q) & 1)) continue;
        const u64x2 d = draw(seed, QSIM_TAG_PAULI, model->epoch, (uint32_t)q);
        const double u = u01(d.a);
        const double p = model->p;
        const int which = u < p / 3.0 ? 1 : u < 2.0 * p / 3.0 ? 2 : u < p ? 3 : 0;
        if (!which) continue;
        double2 P[4];
        if (which == 1) { P[0] = make_double2(0, 0); P[1] = make_double2(1, 0); P[2] = make_double2(1, 0); P[3] = make_double2(0, 0); }
        else if (which == 2) { P[0] = make_double2(0, 0); P[1] = make_double2(0, -1); P[2] = make_double2(0, 1); P[3] = make_double2(0, 0); }
        else { P[0] = make_double2(1, 0); P[1] = make_double2(0, 0); P[2] = make_double2(0, 0); P[3] = make_double2(-1, 0); }
        if (int rc = apply_gate(R, 0, 0, q, P)) return lift(h, R, rc);
        if (ev && count < cap) {
            ev[count].epoch = model->epoch;
            ev[count].qubit = q;
            ev[count].pauli = which;
            ev[count].traj = 0;
        }
        ++count;
    }
    if (nev) *nev = count;
    if (ev && count > cap) return fail(h, QSIM_ERANGE, "event buffer too small");
    return QSIM_OK;
}

// ----------------------------------------------------------------- batched trajectories
int qsim_set_batch(qsim_t *h, int b)
{
    QS_CHECK_HANDLE(h);
    if (b < 0 || b > 24 || b >= h->n) return fail(h, QSIM_ERANGE, "batch bits outside [0, min(n, 25))");
    if (b > 0 && b < h->kglob) return fail(h, QSIM_EINVAL, "the trajectory index must cover the rank bits");
    if (b > 0 && h->n - b < 9) return fail(h, QSIM_ERANGE, "a batched register needs >= 9 qubits");
    const Ranks R = ranks_of(h);
    if (int rc = flush_all(R)) return lift(h, R, rc);
    h->batch_b = b;
    for (Handle *m : R) m->batch_b = b;
    return QSIM_OK;
}

int qsim_batch_set_state(qsim_t *h, const qsim_c128 *reg)
{
    QS_CHECK_HANDLE(h);
    if (!reg) return QSIM_EINVAL;
    if (!h->batch_b) return fail(h, QSIM_EINVAL, "not a batched handle (qsim_set_batch)");
    const Ranks R = ranks_of(h);
    if (int rc = flush_all(R)) return lift(h, R, rc);
    const int r = h->n - h->batch_b;
    const double scale = 1.0 / std::sqrt((double)(1ull << h->batch_b));
    for (Handle *m : R) {
        cudaSetDevice(m->device);
        for (int q = 0; q < m->n; ++q) m->pos[q] = m->n - 1 - q;   // the whole state is overwritten
        double2 *src = nullptr;
        int rc = check_cuda(m, cudaMalloc(&src, sizeof(double2) << r), "batch register buffer");
        if (!rc) rc = check_cuda(m, cudaMemcpyAsync(src, reg, sizeof(double2) << r, cudaMemcpyHostToDevice, m->stream), "batch set state");
        if (!rc) {
            launch_batch_broadcast(m, src, r, scale);
            rc = after_launch(m, "batch broadcast");
        }
        if (!rc) rc = check_cuda(m, cudaStreamSynchronize(m->stream), "batch set state");
        if (src) cudaFree(src);
        if (rc) return lift(h, R, rc);
    }
    return QSIM_OK;
}

int qsim_batch_overlap(qsim_t *h, const qsim_c128 *ref, qsim_c128 *out)
{
    QS_CHECK_HANDLE(h);
    if (!ref || !out) return QSIM_EINVAL;
    if (!h->batch_b) return fail(h, QSIM_EINVAL, "not a batched handle (qsim_set_batch)");
    const Ranks R = ranks_of(h);
    if (int rc = dist_canonicalize(R)) return lift(h, R, rc);
    const int r = h->n - h->batch_b;
    const uint64_t B = 1ull << h->batch_b;
    std::vector<std::vector<double>> parts(R.size(), std::vector<double>(2 * B, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *m = R[i];
        cudaSetDevice(m->device);
        const uint64_t nt = m->local_dim() >> r;
        const uint64_t t0 = ((uint64_t)m->rank << m->nl) >> r;   // canonical: shard = a block of trajectories
        double2 *src = nullptr;
        double *d_out = nullptr;
        int rc = check_cuda(m, cudaMalloc(&src, sizeof(double2) << r), "overlap buffer");
        if (!rc) rc = check_cuda(m, cudaMalloc(&d_out, 2 * nt * sizeof(double)), "overlap buffer");
        if (!rc) rc = check_cuda(m, cudaMemcpyAsync(src, ref, sizeof(double2) << r, cudaMemcpyHostToDevice, m->stream), "overlap");
        if (!rc) {
            launch_batch_overlap(m, src, r, std::sqrt((double)B), d_out);
            rc = after_launch(m, "batch overlap");
        }
        if (!rc) rc = check_cuda(m, cudaMemcpyAsync(parts[i].data() + 2 * t0, d_out, 2 * nt * sizeof(double), cudaMemcpyDeviceToHost, m->stream), "overlap");
        if (!rc) rc = check_cuda(m, cudaStreamSynchronize(m->stream), "overlap");
        if (src) cudaFree(src);
        if (d_out) cudaFree(d_out);
        if (rc) return lift(h, R, rc);
    }
    return lift(h, R, dist_sum_host(R, parts, reinterpret_cast<double *>(out), 2 * B));
}

// ----------------------------------------------------------------- read-out
int qsim_norm(qsim_t *h, double *out)
{
    QS_CHECK_HANDLE(h);
    if (!out) return QSIM_EINVAL;
    return global_norm(h, ranks_of(h), out);
}

int qsim_probs(qsim_t *h, int lo, int m, double *out)
{
    QS_CHECK_HANDLE(h);
    if (!out) return QSIM_EINVAL;
    if (lo < 0 || m < 1 || m > 26 || lo + m > h->n) return fail(h, QSIM_ERANGE, "range outside [0, n) or m > 26");
    const Ranks R = ranks_of(h);
    if (int rc = dist_canonicalize(R)) return lift(h, R, rc);
    // canonical: value bit b <-> position n-lo-m+b; local part [pl, min(nl, pl+m))
    const int nl = h->nl;
    const int pl = h->n - lo - m;
    const int ph = pl + m;   // exclusive
    const uint64_t ny = 1ull << m;
    const int mloc = ph <= nl ? m : (pl < nl ? nl - pl : 0);
    const uint64_t nyl = 1ull << mloc;
    std::vector<std::vector<double>> parts;
    if (R.size() > 1 || mloc != m) parts.assign(R.size(), std::vector<double>(ny, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *hm = R[i];
        cudaSetDevice(hm->device);
        if (hm->probs_cap < nyl) {
            if (hm->d_probs) {
                cudaStreamSynchronize(hm->stream);
                cudaFree(hm->d_probs);
            }
            hm->d_probs = nullptr;
            hm->probs_cap = 0;
            if (cudaMalloc(&hm->d_probs, nyl * sizeof(double)) != cudaSuccess) {
                cudaGetLastError();
                return fail(h, QSIM_ENOMEM, "probs buffer");
            }
            hm->probs_cap = nyl;
        }
        double *d_res = hm->d_probs;
        if (mloc > 0) launch_probs_contig(hm, pl, mloc, d_res);
        else launch_norm(hm, d_res);
        int rc = after_launch(hm, "probs");
        ensure_hred(hm, nyl);   // pinned staging: a pageable D2H of 2^m doubles is several times slower
        if (!rc && !hm->h_red) rc = fail(hm, QSIM_ENOMEM, "pinned probs buffer");
        if (!rc) rc = check_cuda(hm, cudaMemcpyAsync(hm->h_red, d_res, nyl * sizeof(double), cudaMemcpyDeviceToHost, hm->stream), "probs");
        if (!rc) rc = check_cuda(hm, cudaStreamSynchronize(hm->stream), "probs");
        const double *part = hm->h_red;
        if (rc) return lift(h, R, rc);
        if (R.size() == 1 && mloc == m) {
            // one shard holds the whole range: the pinned staging is the result
            std::memcpy(out, part, ny * sizeof(double));
            return QSIM_OK;
        }
        // y = (rank bits inside the range) << mloc | y_loc
        uint64_t yhi = 0;
        if (ph > nl) {
            const int gl = pl > nl ? pl - nl : 0;
            const int gh = ph - nl;
            yhi = ((uint64_t)hm->rank >> gl) & ((1ull << (gh - gl)) - 1);
        }
        for (uint64_t y = 0; y < nyl; ++y) parts[i][(yhi << mloc) | y] = part[y];
    }
    return lift(h, R, dist_sum_host(R, parts, out, ny));
}

int qsim_measure_range(qsim_t *h, int lo, int m, double r, int collapse, uint64_t *y)
{
    QS_CHECK_HANDLE(h);
    if (!y) return QSIM_EINVAL;
    if (lo < 0 || m < 1 || m > 26 || lo + m > h->n) return fail(h, QSIM_ERANGE, "range outside [0, n) or m > 26");
    const uint64_t ny = 1ull << m;
    std::vector<double> P(ny);
    if (int rc = qsim_probs(h, lo, m, P.data())) return rc;   // canonical layout from here on
    // R31: the sequential scan of PAPER.md:400-401 over the marginal
    double acc = 0.0;
    uint64_t v = ny, last_nz = 0;
    for (uint64_t k = 0; k < ny; ++k) {
        if (P[k] > 0.0) last_nz = k;
        acc += P[k];
        if (r < acc) {
            v = k;
            break;
        }
    }
    if (v == ny) v = last_nz;
    *y = v;
    if (!collapse) return QSIM_OK;
    if (!(P[v] > 0.0)) return fail(h, QSIM_ESTATE, "measured value has zero probability (zero state)");
    const double s = 1.0 / std::sqrt(P[v]);
    // canonical: sub-register value bit b <-> position n-lo-m+b; positions >= nl are rank bits
    const Ranks R = ranks_of(h);
    const int pl = h->n - lo - m;
    for (Handle *hm : R) {
        cudaSetDevice(hm->device);
        uint64_t mask = 0, val = 0;
        int zero_all = 0;
        for (int b = 0; b < m; ++b) {
            const int p = pl + b;
            const uint64_t want = (v >> b) & 1;
            if (p < hm->nl) {
                mask |= 1ull << p;
                val |= want << p;
            } else if ((((uint64_t)hm->rank >> (p - hm->nl)) & 1) != want) {
                zero_all = 1;
            }
        }
        launch_collapse(hm, mask, val, s, zero_all);
        if (int rc = after_launch(hm, "collapse")) return lift(h, R, rc);
    }
    return QSIM_OK;
}

int qsim_inner(qsim_t *a, qsim_t *b, qsim_c128 *out)
{
    QS_CHECK_HANDLE(a);
    QS_CHECK_HANDLE(b);
    if (!out) return QSIM_EINVAL;
    const Ranks Ra = ranks_of(a), Rb = ranks_of(b);
    if (a->n != b->n || Ra.size() != Rb.size() || a->world != b->world)
        return fail(a, QSIM_EINVAL, "inner product of registers of different shapes");
    for (size_t i = 0; i < Ra.size(); ++i)
        if (Ra[i]->device != Rb[i]->device || Ra[i]->rank != Rb[i]->rank)
            return fail(a, QSIM_EINVAL, "inner product of registers on different devices");
    if (int rc = dist_canonicalize(Ra)) return lift(a, Ra, rc);
    if (int rc = dist_canonicalize(Rb)) return lift(b, Rb, rc);
    std::vector<std::vector<double>> parts(Ra.size(), std::vector<double>(2, 0.0));
    for (size_t i = 0; i < Ra.size(); ++i) {
        Handle *ha = Ra[i], *hb = Rb[i];
        cudaSetDevice(ha->device);
        // b's shard must be complete before a's stream reads it
        cudaEvent_t ev;
        cudaSetDevice(hb->device);   // the event lives on b's device
        if (int rc = check_cuda(hb, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "inner")) return lift(a, Ra, rc);
        cudaEventRecord(ev, hb->stream);
        cudaSetDevice(ha->device);
        cudaStreamWaitEvent(ha->stream, ev, 0);
        double *d_out = nullptr;
        int rc = check_cuda(ha, cudaMalloc(&d_out, 2 * sizeof(double)), "inner buffer");
        if (!rc) {
            launch_inner(ha, ha->psi, hb->psi, d_out);
            rc = after_launch(ha, "inner");
        }
        if (!rc) rc = check_cuda(ha, cudaMemcpyAsync(parts[i].data(), d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, ha->stream), "inner");
        if (!rc) rc = check_cuda(ha, cudaStreamSynchronize(ha->stream), "inner");
        if (d_out) cudaFree(d_out);
        cudaEventDestroy(ev);
        if (rc) return lift(a, Ra, rc);
    }
    double res[2];
    if (int rc = dist_sum_host(Ra, parts, res, 2)) return lift(a, Ra, rc);
    out->re = res[0];
    out->im = res[1];
    return QSIM_OK;
}

int qsim_prob_index(qsim_t *h, uint64_t idx, double *out)
{
    QS_CHECK_HANDLE(h);
    if (!out) return QSIM_EINVAL;
    if (h->n < 64 && idx >> h->n) return fail(h, QSIM_ERANGE, "index >= 2^n");
    const Ranks R = ranks_of(h);
    if (int rc = dist_canonicalize(R)) return lift(h, R, rc);
    std::vector<std::vector<double>> parts(R.size(), std::vector<double>(1, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *m = R[i];
        cudaSetDevice(m->device);
        if ((int)(idx >> m->nl) != m->rank) continue;
        double2 a;
        if (int rc = check_cuda(m, cudaMemcpyAsync(&a, m->psi + (idx & (m->local_dim() - 1)), sizeof a,
                                                   cudaMemcpyDeviceToHost, m->stream), "prob_index"))
            return lift(h, R, rc);
        if (int rc = check_cuda(m, cudaStreamSynchronize(m->stream), "prob_index")) return lift(h, R, rc);
        parts[i][0] = a.x * a.x + a.y * a.y;
    }
    return lift(h, R, dist_sum_host(R, parts, out, 1));
}

int qsim_measure(qsim_t *h, double r, uint64_t *idx)
{
    QS_CHECK_HANDLE(h);
    if (!idx) return QSIM_EINVAL;
    if (!(r >= 0.0 && r < 1.0)) return fail(h, QSIM_EINVAL, "r must be in [0, 1)");
    const Ranks R = ranks_of(h);
    if (int rc = dist_canonicalize(R)) return lift(h, R, rc);
    const int nl = h->nl;
    const int bb = nl < 16 ? nl : 16;
    const uint64_t nb = (1ull << nl) >> bb;
    const uint64_t total = nb * h->world;
    // block sums of every rank, placed at the rank's blocks
    std::vector<std::vector<double>> parts(R.size(), std::vector<double>(total, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *m = R[i];
        cudaSetDevice(m->device);
        double *d_blk = nullptr;
        if (cudaMalloc(&d_blk, nb * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            return fail(h, QSIM_ENOMEM, "measure buffer");
        }
        launch_block_abs2(m, bb, d_blk);
        int rc = after_launch(m, "measure");
        if (!rc) rc = check_cuda(m, cudaMemcpyAsync(parts[i].data() + nb * m->rank, d_blk, nb * sizeof(double),
                                                    cudaMemcpyDeviceToHost, m->stream), "measure");
        if (!rc) rc = check_cuda(m, cudaStreamSynchronize(m->stream), "measure");
        cudaFree(d_blk);
        if (rc) return lift(h, R, rc);
    }
    std::vector<double> blk(total);
    if (int rc = dist_sum_host(R, parts, blk.data(), total)) return lift(h, R, rc);
    // sequential scan over block sums (fixed order), then inside one block (R22)
    double acc = 0.0;
    int64_t sel = -1, last_nz_blk = -1;
    for (uint64_t b = 0; b < total; ++b) {
        if (blk[b] != 0.0) last_nz_blk = (int64_t)b;
        if (r < acc + blk[b]) { sel = (int64_t)b; break; }
        acc += blk[b];
    }
    const uint64_t blen = 1ull << bb;
    bool fallback = false;
    if (sel < 0) {
        for (uint64_t b = 0; b < total; ++b) if (blk[b] != 0.0) last_nz_blk = (int64_t)b;
        sel = last_nz_blk < 0 ? 0 : last_nz_blk;
        fallback = true;
    }
    const int owner = (int)(((uint64_t)sel * blen) >> nl);
    std::vector<std::vector<double>> res(R.size(), std::vector<double>(1, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *m = R[i];
        cudaSetDevice(m->device);
        if (m->rank != owner) continue;
        std::vector<double2> amp(blen);
        const uint64_t loc = ((uint64_t)sel * blen) & (m->local_dim() - 1);
        int rc = check_cuda(m, cudaMemcpyAsync(amp.data(), m->psi + loc, blen * sizeof(double2), cudaMemcpyDeviceToHost, m->stream), "measure");
        if (!rc) rc = check_cuda(m, cudaStreamSynchronize(m->stream), "measure");
        if (rc) return lift(h, R, rc);
        uint64_t last_nz = 0, result = 0;
        bool found = false;
        double a2 = acc;
        for (uint64_t k = 0; k < blen; ++k) {
            const double p = amp[k].x * amp[k].x + amp[k].y * amp[k].y;
            if (p != 0.0) last_nz = k;
            a2 += p;
            if (!fallback && r < a2) { result = k; found = true; break; }
        }
        if (!found) result = last_nz;
        res[i][0] = (double)(result + (uint64_t)sel * blen);
    }
    double v = 0.0;
    if (int rc = dist_sum_host(R, res, &v, 1)) return lift(h, R, rc);
    *idx = (uint64_t)v;
    return QSIM_OK;
}

// ----------------------------------------------------------------- Shor, semantic mode
static uint64_t host_powmod_u(uint64_t x, uint64_t e, uint64_t N)
{
    unsigned __int128 r = 1 % N, b = x % N;
    for (; e; e >>= 1) {
        if (e & 1) r = r * b % N;
        b = b * b % N;
    }
    return (uint64_t)r;
}

int qsim_shor_semantic_state(qsim_t *h, uint64_t x, uint64_t N, uint64_t v)
{
    QS_CHECK_HANDLE(h);
    if (N < 3 || (N >> 32)) return fail(h, QSIM_ERANGE, "modulus must be in [3, 2^32)");
    if (x >= N || v >= N) return fail(h, QSIM_EINVAL, "x and v must be < N");
    const Ranks R = ranks_of(h);
    std::vector<std::vector<double>> parts(R.size(), std::vector<double>(1, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
        Handle *m = R[i];
        cudaSetDevice(m->device);
        m->queue.clear();   // the state is overwritten
        for (int q = 0; q < m->n; ++q) m->pos[q] = m->n - 1 - q;
        ensure_red(m, 1);
        unsigned long long *d_cnt = reinterpret_cast<unsigned long long *>(m->d_red);
        int rc = check_cuda(m, cudaMemsetAsync(d_cnt, 0, sizeof *d_cnt, m->stream), "shor count");
        if (!rc) {
            launch_shor_count(m, x, N, v, d_cnt);
            rc = after_launch(m, "shor count");
        }
        unsigned long long c = 0;
        if (!rc) rc = check_cuda(m, cudaMemcpyAsync(&c, d_cnt, sizeof c, cudaMemcpyDeviceToHost, m->stream), "shor count");
        if (!rc) rc = check_cuda(m, cudaStreamSynchronize(m->stream), "shor count");
        if (rc) return lift(h, R, rc);
        parts[i][0] = (double)c;   // < 2^53: exact
    }
    double total = 0.0;
    if (int rc = dist_sum_host(R, parts, &total, 1)) return lift(h, R, rc);
    if (total == 0.0) return fail(h, QSIM_EINVAL, "no exponent a < 2^n with x^a = v (mod N)");
    for (Handle *m : R) {
        launch_shor_write(m, x, N, v, 1.0 / std::sqrt(total));
        if (int rc = after_launch(m, "shor state")) return lift(h, R, rc);
    }
    return QSIM_OK;
}

// Post-processing of one measured y (PAPER.md:851-859 steps 4-5; with
// `improved` the four checks of PAPER.md:969-998 in the paper's order, each
// run only when the earlier ones did not finish the iteration -- DESIGN.md
// R27).  mem keeps the candidates of earlier iterations for the LCM Check;
// st accumulates the Table 6 tallies (QSIM_SHOR_*).
static uint64_t shor_postprocess(uint64_t N, uint64_t x, uint64_t y, int nbits, bool improved,
                                 std::vector<uint64_t> &mem, int64_t *st)
{
    const uint64_t M = 1ull << nbits;
    uint64_t cand[64];
    int nc = y ? qsim_shor_candidates(y, nbits, N, cand, 64) : 0;
    if (nc == 0) {
        if (!improved) return 0;
        const int64_t shifts[4] = {1, -1, 2, -2};     // Neighbor y Check
        for (int s = 0; s < 4 && nc == 0; ++s) {
            const int64_t yy = (int64_t)y + shifts[s];
            if (yy > 0 && (uint64_t)yy < M) nc = qsim_shor_candidates((uint64_t)yy, nbits, N, cand, 64);
        }
        st[nc ? QSIM_SHOR_NEIGHBOR_S : QSIM_SHOR_NEIGHBOR_F]++;
        if (nc == 0) return 0;
    }
    const uint64_t r = cand[nc - 1];
    uint64_t f = qsim_shor_try(N, x, r, 0);
    st[f ? QSIM_SHOR_BASIC_S : QSIM_SHOR_BASIC_F]++;
    if (f || !improved) return f;
    auto both = [&](uint64_t rr) {
        uint64_t d = qsim_shor_try(N, x, rr, 0);
        return d ? d : qsim_shor_try(N, x, rr, 1);
    };
    if ((r & 1) == 0) {                                // GCD Check
        f = qsim_shor_try(N, x, r, 1);
        st[f ? QSIM_SHOR_GCD_S : QSIM_SHOR_GCD_F]++;
        if (f) return f;
    }
    if (host_powmod_u(x, r, N) != 1) {                 // Small Factor Check
        for (uint64_t k = 2; k <= 8 && !f; ++k) f = both(k * r);
        st[f ? QSIM_SHOR_SF_S : QSIM_SHOR_SF_F]++;
        if (f) return f;
    }
    if (!mem.empty()) {                                // LCM Check
        for (size_t i = 0; i < mem.size() && !f; ++i) f = both(mem[i] / gcd64(mem[i], r) * r);
        st[f ? QSIM_SHOR_LCM_S : QSIM_SHOR_LCM_F]++;
        if (f) return f;
    }
    if (mem.size() < 64) mem.push_back(r);
    return 0;
}

int qsim_shor_run(qsim_t *h, uint64_t N, uint64_t seed, uint64_t run, int improved, int max_iter,
                  uint64_t *factor, int *iters, int64_t *stats)
{
    int64_t local[QSIM_SHOR_NSTATS] = {0};
    int64_t *st = stats ? stats : local;
    QS_CHECK_HANDLE(h);
    if (!factor || !iters || max_iter < 0) return QSIM_EINVAL;
    *factor = 0;
    *iters = 0;
    if (N < 3 || (N >> 32)) return fail(h, QSIM_ERANGE, "modulus must be in [3, 2^32)");
    const int n = h->n;
    if (n > 62 || (unsigned __int128)N * N > ((unsigned __int128)1 << n))
        return fail(h, QSIM_ERANGE, "exponent register needs 2^n >= N^2 (PAPER.md:841-843)");
    std::vector<uint64_t> mem;
    for (int t = 1; t <= max_iter; ++t) {
        const u64x2 d = draw(seed, QSIM_TAG_SHOR, run, (uint32_t)(t - 1));
        const uint64_t x = 1 + uint_below(d.a, N - 1);
        const uint64_t g = gcd64(x, N);
        if (g > 1 && g < N) {   // step 2
            st[QSIM_SHOR_STEP2]++;
            *factor = g;
            *iters = t;
            return QSIM_OK;
        }
        st[QSIM_SHOR_QUANTUM]++;
        const uint64_t v = host_powmod_u(x, uint_below(d.b, 1ull << n), N);
        if (int rc = qsim_shor_semantic_state(h, x, N, v)) return rc;
        if (int rc = qsim_qft(h, 0, n, 0)) return rc;
        const u64x2 dm = draw(seed, QSIM_TAG_MEASURE, run, (uint32_t)(t - 1));
        uint64_t y = 0;
        if (int rc = qsim_measure(h, u01(dm.a), &y)) return rc;
        if (const uint64_t f = shor_postprocess(N, x, y, n, improved != 0, mem, st)) {
            *factor = f;
            *iters = t;
            return QSIM_OK;
        }
    }
    return QSIM_OK;
}

}  // extern "C"
