// qsim_internal.h -- the handle, layout map and kernel launchers of libqsim.
//
// Layout of the state in HBM: each rank holds one contiguous
// shard of 2^nl complex128 amplitudes (double2: re, im interleaved, 16 B).
// Physical bit positions 0..nl-1 index inside the shard; positions
// nl..n-1 are the rank bits ("global" positions).  The handle keeps a map
// pos[q] = physical position of logical qubit q; the canonical map is
// pos[q] = n-1-q (qubit 0 = MSB).  Kernels only ever see local
// positions; the API layer translates logical qubits through pos[] and
// brings global qubits local with NCCL exchanges (dist.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/qsim.h"

#ifndef QSIM_NO_NCCL
#include <nccl.h>
#endif

namespace qs {

constexpr int kMaxQubits = 40;

constexpr int kMaxFixedBits = 48;

struct Handle;

// --------------------------------------------------------------- kernels
// Every launcher enqueues on h->stream and bumps h->launches.

// Dense 2x2 on local position p; applied where (i & cmask) == cval (local mask).
void launch_apply_2x2(Handle *h, int p, uint64_t cmask, uint64_t cval, const double2 U[4]);
// 2x2 on a rank-bit qubit from the partner's shard over peer memory (out != psi):
// out_i = a psi_i + c theirs_i where (i & cmask) == cval, psi_i elsewhere.
void launch_apply_2x2_remote(Handle *h, const double2 *theirs, double2 *out, uint64_t cmask, uint64_t cval, double2 a,
                             double2 c);
// Diagonal diag(d0, d1) on local position p (both entries applied), controlled.
void launch_apply_diag(Handle *h, int p, uint64_t cmask, uint64_t cval, double2 d0, double2 d1);
// Multiply every amplitude with (i & mask) == val by ph.
void launch_phase_mask(Handle *h, uint64_t mask, uint64_t val, double2 ph);
// Swap local positions p1 != p2.
void launch_swap_local(Handle *h, int p1, int p2);
// Scale every amplitude by s (real).
void launch_scale(Handle *h, double s);
// |0..0> style initialisation: zero the shard, then set element idx (local) to 1.
void launch_zero(Handle *h);
void launch_set_one(Handle *h, uint64_t local_idx);
// Gaussian amplitudes for the shard; logical index of local element i is
// (rank << nl) | i in canonical layout.
void launch_init_gaussian(Handle *h, uint64_t seed);
// sum |a|^2 over the shard -> one double on the device (d_out), tree order.
void launch_norm(Handle *h, double *d_out);
// <a|b> over one shard (a, b: 2^nl amplitudes on this device) -> d_out[0..1]
// (re, im) on the device; fixed tree order.  d_out must not be in the
// reduction workspace.
void launch_inner(Handle *h, const double2 *a, const double2 *b, double *d_out);
// sum of the amplitudes over one shard -> d_out[0..1] (re, im) on the device;
// fixed tree order.  d_out must not be in the reduction workspace.
void launch_amp_sum(Handle *h, double *d_out);
// psi[i] <- c - psi[i] (Grover's diffusion with c = 2 mean).
void launch_reflect(Handle *h, double2 c);
// psi[i] *= s where (i & mask) == val, 0 elsewhere (everywhere if zero_all).
void launch_collapse(Handle *h, uint64_t mask, uint64_t val, double s, int zero_all);
// Partial sums of |a|^2 over consecutive blocks of 2^blk_bits amplitudes.
void launch_block_abs2(Handle *h, int blk_bits, double *d_out);
// Marginals over the `m` physical positions [pl, pl+m) (value bit b <-> position pl+b).
void launch_probs_contig(Handle *h, int pl, int m, double *d_out);
// Modular exponentiation / multiplication permutation (out of place).
struct PermDesc {
    int kind;
    int wpos[40], wm;      // work register: value bit b (LSB = 0) at local position wpos[b]
    int epos[40], em;      // exponent register value bits (LSB = 0): local position, or -1 - g for global bit g
    uint64_t cmask, cval;  // local control mask / values
    uint64_t mult, base, modulus;
    const uint32_t *d_table;
    uint64_t rank_bits;    // this rank's global bits (for exponent bits that are global)
};
int launch_perm(Handle *h, const PermDesc &d);   // QSIM_ENOMEM: the generic path found no scratch
// Grover: iters fused iterations; d_trace receives |a_mark|^2 per iteration.
void launch_grover(Handle *h, uint64_t mark_local, int mark_rank, int iters, double *d_trace);
// Shor semantic-mode register (k_shor.cu): count / write {a : x^a = v mod N}
void launch_shor_count(Handle *h, uint64_t x, uint64_t N, uint64_t v, unsigned long long *d_count);
void launch_shor_write(Handle *h, uint64_t x, uint64_t N, uint64_t v, double amp);

// Fused tile passes (k_tile.cu).  A pass reads every amplitude once and
// writes it once: the shard is cut into tiles of 2^tbits amplitudes that
// share the values of the "fixed" local bits; a CTA gathers a tile (tile bit
// b at input position in_pos[b]), applies the pass's QFT block in registers
// (16 amplitudes per thread, shared-memory transposes between register
// windows), and scatters it to out_pos[] (a bit permutation of the layout
// folded into the store).  With a = 0 the pass is a pure bit permutation.
constexpr int kTileMaxBits = 12;   // <= 4096 amplitudes = 64 KiB of smem
constexpr int kRegBits = 4;        // 16 amplitudes per thread
constexpr int kMaxMaps = 6;

struct TileMap {
    int win[kRegBits];             // tile bits held in registers (slot bit b <-> tile bit win[b])
    int order[kTileMaxBits];       // thread bit t <-> tile bit order[t]
    int ustart, ucnt;              // active wires u in [ustart, ustart+ucnt) get phase + H here
};

struct TilePass {
    int tbits;                     // tile bits (kRegBits+5 <= tbits <= kTileMaxBits)
    int a;                         // active wires: tile bits 0..a-1 in H order (a <= 10)
    int in_pos[kTileMaxBits];      // tile bit -> input local position
    int out_pos[kTileMaxBits];     // tile bit -> output local position
    int nfix;                      // fixed bits: tile index bit f of the tile id
    int fin_pos[kMaxFixedBits];
    int fout_pos[kMaxFixedBits];
    int nmaps;
    TileMap map[kMaxMaps];
    // twiddle exp(+-2 pi i Y J / 2^W): J = sum_u b_u 2^(a-1-u), Y = early-wire value
    int n_et, et_bit[kTileMaxBits], et_w[kTileMaxBits];   // early wires on tile bits
    int n_ef, ef_bit[kMaxFixedBits], ef_w[kMaxFixedBits]; // early wires on fixed bits
    uint64_t y_const;              // early wires on rank bits
    int W;
    int inverse;
    int hadamard_only;             // 1: H on the active wires only (no R_d phases, no twiddle)
    double scale;                  // 2^(-a/2)
    // derived by launch_tile_pass
    uint32_t wswz[kMaxMaps][kRegBits];   // swizzled smem index of each window bit
    uint32_t jwin[kRegBits];             // J weight of the map-0 window bits
    int twiddle_fast;                    // early tile bits are all thread bits of map 0
    double tw;                           // +-2 pi / 2^W
};
// in -> out (may alias when the pass does not move fixed bits between tiles)
void launch_tile_pass(Handle *h, const TilePass &tp, const double2 *in, double2 *out);
// host planner helpers (k_tile.cu): fill tp.map[] from tbits/a/in_pos/out_pos;
// derived constants (swizzle masks, twiddle weights)
void plan_tile_maps(TilePass &tp);
void finish_tile_pass(TilePass &tp);
// TMA-pipelined variant (k_tma.cu); false = geometry unsupported, nothing launched
bool launch_tile_pass_tma(Handle *h, const TilePass &tp, const double2 *in, double2 *out);

// Generalised QFT pass (k_tma.cu k_qft_gen): the same block structure with
// arbitrary per-gate data -- the noisy H matrices and R_d angles of a circuit
// with operational error or the R_d of an approximate QFT
// left out.  Active wire u (tile bit u) of the pass:
// before its H, the amplitudes with b_u = 1 get exp(i (hph[u] + sum_{earlier
// wires i, y_i = 1} phe[u][i])) (H's column phase and the earlier blocks: a
// twiddle per tile) times prod_{u' < u, b_u' = 1} ein[u][u'] (this block);
// then the real 2x2 Hr[u].  Every H of the paper's circuits has this form:
// U_R(t) U_P1(p) = [[c, -s e^{ip}], [s, c e^{ip}]] and the
// exact H (t = pi/4, p = pi) with the phase folded into the real part.
// phe[u][i] = angle of R(a0+u, i), ein[u][u'] = e^{i angle of R(a0+u, a0+u')}.
constexpr int kGenWires = 10;
constexpr int kGenEarly = 48;
struct QftGen {
    double Hr[kGenWires][4];
    double hph[kGenWires];
    double2 ein[kGenWires][kGenWires];
    double phe[kGenWires][kGenEarly];
};
// true: launched; false: the pass geometry does not fit the kernel (nothing launched)
bool launch_qft_gen_tma(Handle *h, const TilePass &tp, const QftGen &g, const double2 *in, double2 *out);

// A fused QFT / H pass on 2^13-amplitude tiles (k_qft13.cu): tile bits 0..a-1
// are the active wires in H order, a..12 passive positions; same twiddle
// fields as TilePass.  Fixed positions fin_pos[] must be ascending (tile-id
// bit f <-> the f-th lowest fixed position).  false: geometry unsupported.
constexpr int kTile13Bits = 13;
struct Qft13Desc {
    int a;
    int in_pos[kTile13Bits], out_pos[kTile13Bits];
    int nfix;
    int fin_pos[kMaxFixedBits], fout_pos[kMaxFixedBits];
    int n_et, et_bit[kTile13Bits], et_w[kTile13Bits];
    int n_ef, ef_bit[kMaxFixedBits], ef_w[kMaxFixedBits];
    uint64_t y_const;
    int W, inverse, hadamard_only;
    double scale;
    // rank-group pass (api.cu fused_range, in-process groups): ng <= 2 tile
    // bits gbit[] (ascending position) sit on rank bits (in_pos >= nl, out_pos
    // -1); the pass runs in place on the 2^ng shards gbase[c] (c = the global
    // bits' values) and this rank takes the tiles whose tile-id bits
    // split_fix[] (ascending) equal split_val's bits
    int ng;
    int gbit[2], split_fix[2];
    uint64_t split_val;
    double2 *gbase[4];
};
bool launch_qft13(Handle *h, const Qft13Desc &d, const double2 *in, double2 *out);
bool qft_gen_feasible(Handle *h, const TilePass &tp);

// Fused gate-list passes (k_ops.cu): ops of one pass, applied per tile.
// Op kinds (encoded per segment on the host, so the kernel's per-op work is
// a few uniform tests and statically indexed register updates):
//   DENSE   2x2 on window bit rb          DIAGW  diag(d0, d1) on window bit rb
//   DIAGT   diag on a thread-part bit     DIAGF  diag on a fixed (tile-id) bit
//   PHASE   constant phase u[3]
//   CDENSE  2x2 on window bit rb where window bit cs == cv (one control)
//   DENSE2  2x2 on window bit rb: u[0..3] where window bit cs = 0, u[4..7]
//           where it is 1 (a run of gates on one target, each uncontrolled or
//           controlled by the same qubit, multiplied together on the host);
//           DENSE with tsel / fsel is the same choice by a thread-part or a
//           tile-id bit (one matrix per thread / per tile: no divergence)
//   DENSET  2x2 on window bit rb with one matrix per trajectory of a batched
//           handle (batch.cu): tab[4 t .. 4 t + 3], t from the tile id
// Controls: wm/wv on the 4 window bits (slot index), tm/tv on the other tile
// bits (thread part), fm/fv on fixed bits (tile id).
enum { GOP_DENSE = 0, GOP_DIAGW = 1, GOP_DIAGT = 2, GOP_DIAGF = 3, GOP_PHASE = 4, GOP_CDENSE = 5, GOP_DENSE2 = 6,
       GOP_DENSET = 7 };
struct GOp {
    uint8_t kind, rb, wm, wv;
    uint8_t cs, cv;
    uint8_t fsel;      // DENSE: tile-id bit selecting u[4..7] (0xff: none)
    uint8_t pad_;
    uint32_t tm, tv;   // controls on non-window tile bits
    uint32_t tb;       // DIAGT: mask of the target tile bit
    uint32_t fbit;     // DIAGF: tile-id bit of the target
    uint32_t tsel;     // DENSE: thread-part bit selecting u[4..7] (0: none)
    uint32_t code;     // dispatch word (op_code(), plan_ops.cu): case id | kOpChk* flags
    uint64_t fm, fv;   // controls on fixed bits (tile-id mask / values)
    const double2 *tab;   // DENSET: per-trajectory matrices (device memory)
    double2 u[8];      // dense U (u11 u12 u21 u22) or diag(u[0], u[3]); DENSE2: two matrices
};
// GOp::code: bits 0-7 the interpreter's case (ops_common.cuh apply_op), plus
// which run-time checks the op needs
constexpr uint32_t kOpChkFixed = 1u << 8;    // fm / fv
constexpr uint32_t kOpChkThread = 1u << 9;   // tm / tv
constexpr uint32_t kOpSel = 1u << 10;        // tsel / fsel matrix choice
constexpr uint32_t kOpTraj = 1u << 11;       // DENSET: the tile's trajectory matrix from op.tab
enum {
    OPC_DENSE = 0,      // + rb (+5: window controls); DENSET too (kOpTraj)
    OPC_CDENSE = 20,    // + rb*10 + cs*2 + cv
    OPC_DENSE2 = 70,    // + rb*5 + cs
    OPC_DIAGW = 95,     // + rb*4 + 2*(window controls) + (d0 == 1)
    OPC_OTHER = 115     // PHASE / DIAGT / DIAGF
};
constexpr int kMaxSegs = 48;
constexpr int kOpsRegBits = 5;   // gate-list passes: 32 amplitudes per thread
struct OpsSeg {
    int win[kOpsRegBits];       // tile bits held in registers (slot bit b <-> tile bit win[b])
    int order[kTileMaxBits];    // thread bit t <-> tile bit order[t]
    int op_begin, op_end;
};
struct OpsPass {
    int tbits;
    int in_pos[kTileMaxBits];   // tile bit -> local position (in place: same on output)
    int nfix;
    int fin_pos[kMaxFixedBits];
    int nops, nseg;
    // trajectory index of a tile (batched handles): t = t_rank | sum_i bit(T, bat_fix[i]) << bat_sh[i]
    int nbat;
    int bat_fix[24], bat_sh[24];
    uint32_t bat_rank;
    OpsSeg seg[kMaxSegs];
};
// One launch: the pass geometry and its op list travel as one __grid_constant__
// kernel parameter (<= 32 KiB), so every op read is a uniform constant-bank load
// (no shared-memory traffic, no per-handle device buffer).
constexpr int kOpsParam = 136;
struct OpsLaunch {
    OpsPass P;
    GOp ops[kOpsParam];
};
static_assert(sizeof(OpsLaunch) <= 32000, "kernel parameter space");
static_assert(sizeof(GOp) % 16 == 0, "op records are copied to shared memory in 16-byte words");
// k_ops_pp keeps 3 x 64 KiB stages and the op list in one CTA's shared memory (227 KiB opt-in)
static_assert(3 * (16 << kTileMaxBits) + 64 + kOpsParam * sizeof(GOp) <= 232448, "k_ops_pp shared memory");
void launch_ops_pass(Handle *h, const OpsLaunch &L);
bool launch_ops_pass_tma(Handle *h, const OpsLaunch &L);
bool launch_ops_pass_pp(Handle *h, const OpsLaunch &L);   // k_tma.cu ping-pong; false: geometry   // k_tma.cu; false: geometry unsupported

// A queued gate in physical local positions (api.cu gate queue).
struct QOp {
    int diag;          // 1: diagonal (u[1] = u[2] = 0)
    int tpos;          // target local position; -1 for a constant phase (diag only)
    uint64_t cmask, cval;   // controls on local positions
    double2 u[4];
    const double2 *tab = nullptr;   // batched handle: one matrix per trajectory (then u is unused)
};

// --------------------------------------------------------------- handle
struct Handle {
    int n = 0;              // qubits
    int world = 1, rank = 0;
    int kglob = 0;          // log2(world)
    int nl = 0;             // local qubits
    int device = 0;
    cudaStream_t stream = nullptr;
    double2 *psi = nullptr;      // shard (2^nl)
    double2 *scratch = nullptr;  // lazily allocated, 2^nl (bit permutations, exchanges)
    int pos[kMaxQubits];         // logical qubit -> physical position
    // reduction workspace
    double *d_red = nullptr;
    size_t red_cap = 0;          // doubles
    double *d_probs = nullptr;   // qsim_probs output (grow-only)
    size_t probs_cap = 0;
    double *h_red = nullptr;     // pinned
    size_t hred_cap = 0;
    double *d_sum2 = nullptr;    // 2 doubles: amplitude-sum result (diffusion), outside d_red
    // host-stream pipeline (qsim_qft_host_stream): two extra shard buffers and
    // the copy streams (created on first use)
    double2 *stage[2] = {nullptr, nullptr};
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaStream_t s_comm = nullptr;   // shard-exchange stream (dist.cu), created on first use
    int strict = 0;              // qsim_set_strict: reject non-unitary matrices (QSIM_ENONUNITARY)
    // angle noise (R15)
    uint64_t noise_seed = 0;
    double sigma = 0.0;
    uint64_t gcount = 0;
    // bookkeeping
    uint64_t launches = 0;
    int poisoned = 0;
    std::string err;
#ifndef QSIM_NO_NCCL
    ncclComm_t comm = nullptr;
#endif
    int num_sms = 148;
    // profiling
    int prof_on = 0;
    struct ProfRec { const char *name; uint64_t bytes; cudaEvent_t a, b; uint64_t fp64; };
    uint64_t prof_fp64 = 0;   // algorithmic FP64 instructions of the next launch (prof_set_fp64)
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    cudaEvent_t pending = nullptr;
    std::string prof_json;
    // gate queue (fused into k_ops passes at the next flush)
    std::vector<QOp> queue;
    int fuse = 1;
    // batched trajectories (batch.cu, R33): qubits [0, batch_b) index them
    int batch_b = 0;
    double2 *d_tabs = nullptr;   // per-trajectory matrix tables of queued gates (reset at flush)
    size_t tabs_cap = 0, tabs_used = 0;   // in double2
    // multi-process world: peers' shard buffers mapped with CUDA IPC for the
    // fused remote gate (dist.cu), set up on first use (ipc_state: 0 not yet,
    // 1 ready, -1 unavailable)
    int ipc_state = 0;
    double2 *own_buf[2] = {nullptr, nullptr};   // this rank's two allocations (psi / scratch at setup)
    std::vector<double2 *> peer_buf;            // 2 * world: rank r's allocations 0 and 1
    // in-process rank group (qsim_create_group): the group handle owns the
    // member handles (one shard each); members point back at the group
    std::vector<Handle *> members;
    Handle *grp = nullptr;

    uint64_t local_dim() const { return (uint64_t)1 << nl; }
};

// Function attributes (dynamic smem limits) are per device: true the first
// time it is called for the current device (per call site).
inline bool first_use_on_device(uint64_t &mask)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (mask & bit) return false;
    mask |= bit;
    return true;
}

// per-launch profiling (qsim_profile): events around every kernel launch when
// enabled; prof_end also counts the launch.
void prof_begin(Handle *h);
void prof_end(Handle *h, const char *name, uint64_t bytes);
// the algorithmic FP64 instructions (FMA / MUL / ADD, one per lane) of the
// next launch, for FP64-bound kernels' roofline (qsim_profile_json "fp64")
inline void prof_set_fp64(Handle *h, uint64_t n) { h->prof_fp64 = n; }
struct OpsLaunch;
// FP64 instructions of a gate-list pass: 16 per amplitude pair of a dense
// 2x2 (8 per amplitude), 4 per amplitude a phase multiplies, scaled by the
// fraction of amplitudes each op's controls select
uint64_t ops_fp64(const OpsLaunch &L);
void prof_end_comm(Handle *h, const char *name, uint64_t bytes);   // exchanges: bytes sent + received

// error helpers
int fail(Handle *h, int code, const std::string &msg);
int check_cuda(Handle *h, cudaError_t e, const char *what);
void ensure_red(Handle *h, size_t doubles);
void ensure_hred(Handle *h, size_t doubles);
int ensure_scratch(Handle *h);
inline void swap_buffers(Handle *h)
{
    double2 *t = h->psi;
    h->psi = h->scratch;
    h->scratch = t;
}

// The rank shards this process drives: one handle (single GPU, or one rank
// of a multi-process NCCL world), or every member of an in-process group.
using Ranks = std::vector<Handle *>;
inline Ranks ranks_of(Handle *h) { return h->members.empty() ? Ranks{h} : h->members; }

// distributed layer (dist.cu): every step runs on all ranks of R in lock step
int dist_make_local(const Ranks &R, const std::vector<int> &need);   // make logical qubits local
// a non-diagonal gate on a rank-bit qubit in one peer-memory kernel per rank
// (in-process rank groups); false: not available here (use dist_make_local)
bool dist_remote_gate_available(const Ranks &R);
int dist_remote_gate(const Ranks &R, uint64_t cmask, uint64_t cvals, int q, const double2 U[4]);
int dist_canonicalize(const Ranks &R);                               // pos[q] = n-1-q everywhere
// multi-process world: every rank's current shard as a pointer in this
// process (CUDA IPC; 1: not available), and a stream-ordered all-rank barrier
int dist_world_shards(Handle *h, std::vector<double2 *> &shards);
int dist_world_barrier(Handle *h);
// per-rank host partials -> the sum over all ranks of the world, in rank order
// (parts[i] belongs to R[i]); out may alias parts[0]
int dist_sum_host(const Ranks &R, const std::vector<std::vector<double>> &parts, double *out, size_t count);
// batched trajectories (batch.cu)
void launch_batch_mats(Handle *h, int kind, const double *ang, double sigma, uint64_t seed, uint64_t g, uint64_t B,
                       double2 *out);
void launch_batch_broadcast(Handle *h, const double2 *src, int r, double scale);
// out[t] = B_t A_t for trajectories t < count (2x2 complex, row-major); a null
// table means the constant matrix ac / bc for every t (batch.cu)
void launch_batch_mul(Handle *h, double2 *out, const double2 *A, const double2 ac[4], const double2 *B,
                      const double2 bc[4], uint64_t count);
void launch_batch_overlap(Handle *h, const double2 *ref, int r, double scale, double *d_out);
// one queued gate with the unfused streaming kernels (k_gates.cu)
void run_gate_unfused(Handle *h, const QOp &op);
// run every queued gate (fused passes); called before anything that reads or moves data
int flush_queue(Handle *h);
int flush_all(const Ranks &R);
// local bit-permutation pass (api.cu): new position of old local position p is perm[p]
void permute_local(Handle *h, const std::vector<int> &perm);

}  // namespace qs

struct qsim_s : public qs::Handle {};
