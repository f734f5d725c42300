// dist.cu -- state-vector sharding over GPUs (one process per GPU, NCCL).
//
// The paper's "large subblock" rule (§2.2.1): the rows j
// and j + 2^(n-i-1) of a gate on qubit i must meet on one processor.  On P
// GPUs the state is sharded on its top log2(P) physical bits ("global"
// positions nl..n-1 = the rank bits).  A non-diagonal gate on a qubit at a
// global position g first swaps that qubit with the top local position:
// rank r exchanges the half of its shard whose top local bit differs from
// its own bit g with partner r ^ 2^(g-nl) (ncclSend/ncclRecv in one group;
// the half is one contiguous block of S/2 bytes).  Only the logical ->
// physical map changes; nothing is swapped back.  Diagonal gates and
// gates whose controls sit on rank bits need no communication.
//
// Read-outs restore the canonical layout first: global positions by
// pairwise exchanges, local positions by one bit-permutation pass.
// Host-side partial results are combined in fixed rank order (allgather,
// then summed on the host), so results are deterministic.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "qsim_internal.h"

namespace qs {

#ifndef QSIM_NO_NCCL
static int nccl_check(Handle *h, ncclResult_t r, const char *what)
{
    if (r == ncclSuccess) return QSIM_OK;
    h->poisoned = 1;
    return fail(h, QSIM_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
#endif

// Host-side planner (pure; exported as qsim_plan_make_local /
// qsim_plan_canonicalize for the multi-process CPU tests).  A plan is a list
// of steps on the physical layout:
//   {LSWAP, p1, p2}: swap local positions p1 and p2 (a half pass on the shard)
//   {XCHG, g, -}   : swap global position g with the top local position nl-1
//                    (rank r exchanges its half with top bit != bit g of r with
//                    rank r ^ 2^(g-nl))
//   {A2A, k, -}    : swap all k global positions nl..nl+k-1 with the top k
//                    local positions nl-k..nl-1 at once: rank r sends its
//                    block j (top local bits = j) to rank j and receives that
//                    rank's block r -- one all-to-all of (1 - 2^-k) S per rank
//                    instead of k pairwise exchanges of S/2 (SURVEY §8(e) ii)
// and pos[] (logical -> physical) is updated as the steps would move the data.
enum { STEP_LSWAP = 0, STEP_XCHG = 1, STEP_A2A = 2 };
struct Step { int kind, a, b; };

static int qubit_at(const std::vector<int> &pos, int p)
{
    for (int q = 0; q < (int)pos.size(); ++q)
        if (pos[q] == p) return q;
    return -1;
}

static void apply_step(std::vector<int> &pos, int nl, const Step &s)
{
    if (s.kind == STEP_A2A) {
        for (int i = 0; i < s.a; ++i) {
            const int qa = qubit_at(pos, nl - s.a + i), qb = qubit_at(pos, nl + i);
            std::swap(pos[qa], pos[qb]);
        }
        return;
    }
    const int pa = s.a, pb = s.kind == STEP_LSWAP ? s.b : nl - 1;
    const int qa = qubit_at(pos, pa), qb = qubit_at(pos, pb);
    std::swap(pos[qa], pos[qb]);
}

static int plan_make_local(int n, int nl, std::vector<int> &pos, const std::vector<int> &need,
                           std::vector<Step> &steps, bool allow_a2a = true)
{
    std::vector<char> needed(n, 0);
    for (int q : need) needed[q] = 1;
    const int k = n - nl;
    int nglob = 0;
    for (int q : need) nglob += pos[q] >= nl;
    if (allow_a2a && k >= 2 && nglob >= 2 && nl - k >= 0) {
        // every global qubit local with one all-to-all: first move needed
        // qubits out of the top k local positions (the victims)
        for (int p = nl - k; p < nl; ++p) {
            if (!needed[qubit_at(pos, p)]) continue;
            int dst = -1;
            for (int d = nl - k - 1; d >= 0 && dst < 0; --d)
                if (!needed[qubit_at(pos, d)]) dst = d;
            if (dst < 0) return QSIM_EINVAL;
            steps.push_back({STEP_LSWAP, dst, p});
            apply_step(pos, nl, steps.back());
        }
        steps.push_back({STEP_A2A, k, -1});
        apply_step(pos, nl, steps.back());
        return QSIM_OK;
    }
    for (int q : need) {
        const int g = pos[q];
        if (g < nl) continue;
        // victim: the highest local position holding a qubit we do not need
        int victim = -1;
        for (int p = nl - 1; p >= 0 && victim < 0; --p)
            if (!needed[qubit_at(pos, p)]) victim = p;
        if (victim < 0) return QSIM_EINVAL;
        if (victim != nl - 1) {
            steps.push_back({STEP_LSWAP, victim, nl - 1});
            apply_step(pos, nl, steps.back());
        }
        steps.push_back({STEP_XCHG, g, -1});
        apply_step(pos, nl, steps.back());
    }
    return QSIM_OK;
}

// Global positions to canonical (qubit n-1-g at global position g); the local
// positions are left to one bit-permutation pass.
static int plan_canonical_globals(int n, int nl, std::vector<int> &pos, std::vector<Step> &steps)
{
    for (int g = nl; g < n; ++g) {
        const int want = n - 1 - g;
        if (pos[want] == g) continue;
        if (pos[want] >= nl) {
            // bring it local first (it sits on a global position > g, so the
            // positions already placed are not touched)
            if (int rc = plan_make_local(n, nl, pos, std::vector<int>{want}, steps, false)) return rc;
        }
        const int p = pos[want];
        if (p != nl - 1) {
            steps.push_back({STEP_LSWAP, p, nl - 1});
            apply_step(pos, nl, steps.back());
        }
        steps.push_back({STEP_XCHG, g, -1});
        apply_step(pos, nl, steps.back());
    }
    return QSIM_OK;
}

// ---------------------------------------------------------------- transport
// XCHG g: rank r swaps the half of its shard whose top local bit differs from
// its rank bit g with rank r ^ 2^(g-nl) (whose half has the other top bit),
// so afterwards the qubits at position g and nl-1 have traded places.
//
// Both transports move the half in chunks (QSIM_XCHG_CHUNK_KB, default
// 64 MiB) on two streams so the steps overlap:
//  * multi-process world (one rank per process): chunk c goes out and comes
//    in with ncclSend + ncclRecv in one group on the handle's comm stream
//    (into the scratch shard), and is copied into place on the compute stream
//    as soon as its group completes -- while chunk c+1 is on the wire;
//  * in-process group (qsim_create_group): the lower rank's stream parks its
//    chunk in its scratch and pulls the partner's chunk (peer copies over
//    NVLink between GPUs), the partner's stream writes the parked chunk into
//    its own half, chunk by chunk, ordered by events.

static uint64_t xchg_chunk_amps(uint64_t half)
{
    static const long kb = std::getenv("QSIM_XCHG_CHUNK_KB") ? std::atol(std::getenv("QSIM_XCHG_CHUNK_KB")) : 65536;
    uint64_t c = (uint64_t)(kb > 0 ? kb : 65536) * 1024 / sizeof(double2);
    if (c < 1) c = 1;
    while (half / c > 64) c <<= 1;   // at most 64 chunks
    return c < half ? c : half;
}

static int comm_stream(Handle *h)
{
    if (h->s_comm) return QSIM_OK;
    return check_cuda(h, cudaStreamCreateWithFlags(&h->s_comm, cudaStreamNonBlocking), "comm stream");
}

static int exchange_nccl(Handle *h, int g)
{
#ifndef QSIM_NO_NCCL
    const int gb = g - h->nl;
    const int partner = h->rank ^ (1 << gb);
    const int b = (h->rank >> gb) & 1;
    const uint64_t half = h->local_dim() >> 1;
    if (int rc = ensure_scratch(h)) return rc;
    if (int rc = comm_stream(h)) return rc;
    double2 *mine = h->psi + (uint64_t)(1 - b) * half;
    const uint64_t ca = xchg_chunk_amps(half);
    prof_begin(h);
    cudaEvent_t ready;
    cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    cudaEventRecord(ready, h->stream);
    cudaStreamWaitEvent(h->s_comm, ready, 0);
    cudaEventDestroy(ready);
    for (uint64_t off = 0; off < half; off += ca) {
        const uint64_t cnt = std::min<uint64_t>(ca, half - off);
        if (int rc = nccl_check(h, ncclGroupStart(), "ncclGroupStart")) return rc;
        ncclSend(mine + off, cnt * 2, ncclDouble, partner, h->comm, h->s_comm);
        ncclRecv(h->scratch + off, cnt * 2, ncclDouble, partner, h->comm, h->s_comm);
        if (int rc = nccl_check(h, ncclGroupEnd(), "ncclGroupEnd")) return rc;
        cudaEvent_t done;
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
        cudaEventRecord(done, h->s_comm);
        cudaStreamWaitEvent(h->stream, done, 0);
        cudaEventDestroy(done);
        cudaError_t e = cudaMemcpyAsync(mine + off, h->scratch + off, cnt * sizeof(double2), cudaMemcpyDeviceToDevice,
                                        h->stream);
        if (e != cudaSuccess) return check_cuda(h, e, "exchange copy");
    }
    prof_end_comm(h, "nccl_pair_exchange", half * 32);
    return QSIM_OK;
#else
    (void)g;
    return fail(h, QSIM_ENCCL, "built without NCCL");
#endif
}

static int alltoall_nccl(Handle *h, int k)
{
#ifndef QSIM_NO_NCCL
    const uint64_t blk = h->local_dim() >> k;
    if (int rc = ensure_scratch(h)) return rc;
    if (int rc = comm_stream(h)) return rc;
    prof_begin(h);
    cudaEvent_t ready, done;
    cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    cudaEventRecord(ready, h->stream);
    cudaStreamWaitEvent(h->s_comm, ready, 0);
    if (int rc = nccl_check(h, ncclGroupStart(), "ncclGroupStart")) return rc;
    for (int p = 0; p < h->world; ++p) {
        if (p == h->rank) continue;
        ncclSend(h->psi + (uint64_t)p * blk, blk * 2, ncclDouble, p, h->comm, h->s_comm);
        ncclRecv(h->scratch + (uint64_t)p * blk, blk * 2, ncclDouble, p, h->comm, h->s_comm);
    }
    if (int rc = nccl_check(h, ncclGroupEnd(), "ncclGroupEnd")) return rc;
    cudaEventRecord(done, h->s_comm);
    // this rank's own block moves locally while the others are on the wire
    cudaError_t e = cudaMemcpyAsync(h->scratch + (uint64_t)h->rank * blk, h->psi + (uint64_t)h->rank * blk,
                                    blk * sizeof(double2), cudaMemcpyDeviceToDevice, h->stream);
    cudaStreamWaitEvent(h->stream, done, 0);
    cudaEventDestroy(ready);
    cudaEventDestroy(done);
    prof_end_comm(h, "nccl_alltoall", (uint64_t)(h->world - 1) * blk * 32);
    if (e != cudaSuccess) return check_cuda(h, e, "all-to-all copy");
    swap_buffers(h);
    return QSIM_OK;
#else
    (void)k;
    return fail(h, QSIM_ENCCL, "built without NCCL");
#endif
}

// In-process group: member r pulls block r of every member p into block p of
// its scratch shard (peer copies), ordered after every member's pending work;
// then every member swaps shard and scratch.
static int alltoall_group(const Ranks &R, int k)
{
    const size_t P = R.size();
    const uint64_t blk = R[0]->local_dim() >> k;
    for (Handle *m : R)
        if (int rc = ensure_scratch(m)) return rc;
    std::vector<cudaEvent_t> pre(P), post(P);
    for (size_t i = 0; i < P; ++i) {
        cudaSetDevice(R[i]->device);   // events live on their stream's device
        cudaEventCreateWithFlags(&pre[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&post[i], cudaEventDisableTiming);
        cudaEventRecord(pre[i], R[i]->stream);
    }
    for (size_t r = 0; r < P; ++r) {
        cudaSetDevice(R[r]->device);
        for (size_t m = 0; m < P; ++m) cudaStreamWaitEvent(R[r]->stream, pre[m], 0);
        for (size_t p = 0; p < P; ++p)
            cudaMemcpyAsync(R[r]->scratch + p * blk, R[p]->psi + r * blk, blk * sizeof(double2), cudaMemcpyDefault,
                            R[r]->stream);
        cudaEventRecord(post[r], R[r]->stream);
    }
    for (size_t m = 0; m < P; ++m) {
        cudaSetDevice(R[m]->device);
        for (size_t r = 0; r < P; ++r) cudaStreamWaitEvent(R[m]->stream, post[r], 0);
    }
    for (Handle *m : R) swap_buffers(m);
    for (size_t i = 0; i < P; ++i) {
        cudaEventDestroy(pre[i]);
        cudaEventDestroy(post[i]);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QSIM_OK : check_cuda(R[0], e, "group all-to-all");
}

static int exchange_pair(Handle *A, Handle *B, int g)
{
    (void)g;
    // A = lower rank (bit g = 0): its half with top bit 1 <-> B's half with top bit 0
    const uint64_t half = A->local_dim() >> 1;
    if (int rc = ensure_scratch(A)) return rc;
    double2 *ha = A->psi + half, *hb = B->psi;
    const uint64_t ca = xchg_chunk_amps(half);
    // an event lives on its stream's device (the members may sit on different GPUs)
    cudaEvent_t eb, ea;
    cudaSetDevice(B->device);
    cudaEventCreateWithFlags(&eb, cudaEventDisableTiming);
    cudaEventRecord(eb, B->stream);
    cudaSetDevice(A->device);
    cudaStreamWaitEvent(A->stream, eb, 0);
    prof_begin(A);
    for (uint64_t off = 0; off < half; off += ca) {
        const size_t bytes = std::min<uint64_t>(ca, half - off) * sizeof(double2);
        // A parks its chunk and pulls B's; B then writes the parked chunk into its half
        cudaSetDevice(A->device);
        cudaMemcpyAsync(A->scratch + off, ha + off, bytes, cudaMemcpyDefault, A->stream);
        cudaMemcpyAsync(ha + off, hb + off, bytes, cudaMemcpyDefault, A->stream);
        cudaEventCreateWithFlags(&ea, cudaEventDisableTiming);
        cudaEventRecord(ea, A->stream);
        cudaSetDevice(B->device);
        cudaStreamWaitEvent(B->stream, ea, 0);
        cudaMemcpyAsync(hb + off, A->scratch + off, bytes, cudaMemcpyDefault, B->stream);
        cudaEventDestroy(ea);
    }
    // A's scratch is read by B's copies: A waits for them before reusing it
    cudaSetDevice(B->device);
    cudaEventRecord(eb, B->stream);
    cudaSetDevice(A->device);
    cudaStreamWaitEvent(A->stream, eb, 0);
    prof_end_comm(A, "group_pair_exchange", half * 32);
    cudaSetDevice(B->device);
    cudaEventDestroy(eb);
    cudaSetDevice(A->device);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QSIM_OK : check_cuda(A, e, "group exchange");
}

static int run_steps(const Ranks &R, const std::vector<Step> &steps)
{
    const bool group = R.size() > 1;
    for (const Step &st : steps) {
        if (st.kind == STEP_LSWAP) {
            for (Handle *h : R) launch_swap_local(h, st.a, st.b);
        } else if (st.kind == STEP_A2A) {
            if (group) {
                if (int rc = alltoall_group(R, st.a)) return rc;
            } else {
                if (int rc = alltoall_nccl(R[0], st.a)) return rc;
            }
        } else if (group) {
            const int gb = st.a - R[0]->nl;
            for (size_t r = 0; r < R.size(); ++r) {
                const size_t p = r ^ ((size_t)1 << gb);
                if (r < p)
                    if (int rc = exchange_pair(R[r], R[p], st.a)) return rc;
            }
        } else {
            if (int rc = exchange_nccl(R[0], st.a)) return rc;
        }
        for (Handle *h : R) {
            std::vector<int> pos(h->pos, h->pos + h->n);
            apply_step(pos, h->nl, st);
            for (int q = 0; q < h->n; ++q) h->pos[q] = pos[q];
        }
    }
    return QSIM_OK;
}

// ---------------------------------------------------------------- fused remote gate
#ifndef QSIM_NO_NCCL
// Multi-process world: map every rank's two shard allocations into this
// process (cudaIpcGetMemHandle / OpenMemHandle, handles exchanged with one
// NCCL all-gather).  Collective; all ranks agree on success (min-reduce), so
// either every rank uses the remote path or none does.
static int ipc_setup(Handle *h)
{
    if (h->ipc_state) return h->ipc_state;
    h->ipc_state = -1;
    if (ensure_scratch(h)) return -1;
    h->own_buf[0] = h->psi;
    h->own_buf[1] = h->scratch;
    const int W = h->world;
    const size_t hs = sizeof(cudaIpcMemHandle_t);
    std::vector<unsigned char> mine(2 * hs, 0), all(2 * hs * W, 0);
    int ok = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t *>(mine.data()), h->own_buf[0]) == cudaSuccess &&
             cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t *>(mine.data() + hs), h->own_buf[1]) == cudaSuccess;
    cudaGetLastError();
    unsigned char *d_in = nullptr, *d_out = nullptr;
    int *d_ok = nullptr;
    if (cudaMalloc(&d_in, mine.size()) != cudaSuccess || cudaMalloc(&d_out, all.size()) != cudaSuccess ||
        cudaMalloc(&d_ok, sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;   // still take part in the collectives below
    }
    if (d_in && d_out && d_ok) {
        cudaMemcpyAsync(d_in, mine.data(), mine.size(), cudaMemcpyHostToDevice, h->stream);
        ncclAllGather(d_in, d_out, mine.size(), ncclUint8, h->comm, h->stream);
        cudaMemcpyAsync(all.data(), d_out, all.size(), cudaMemcpyDeviceToHost, h->stream);
        cudaStreamSynchronize(h->stream);
    }
    h->peer_buf.assign(2 * W, nullptr);
    for (int r = 0; r < W && ok; ++r) {
        if (r == h->rank) {
            h->peer_buf[2 * r] = h->own_buf[0];
            h->peer_buf[2 * r + 1] = h->own_buf[1];
            continue;
        }
        for (int k = 0; k < 2 && ok; ++k) {
            cudaIpcMemHandle_t ih;
            std::memcpy(&ih, all.data() + (2 * r + k) * hs, hs);
            void *p = nullptr;
            if (cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                ok = 0;
            }
            h->peer_buf[2 * r + k] = static_cast<double2 *>(p);
        }
    }
    // agree: min over ranks
    if (d_ok) {
        cudaMemcpyAsync(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice, h->stream);
        ncclAllReduce(d_ok, d_ok, 1, ncclInt, ncclMin, h->comm, h->stream);
        cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, h->stream);
        cudaStreamSynchronize(h->stream);
    }
    if (d_in) cudaFree(d_in);
    if (d_out) cudaFree(d_out);
    if (d_ok) cudaFree(d_ok);
    cudaGetLastError();
    h->ipc_state = ok ? 1 : -1;
    return h->ipc_state;
}
#endif

bool dist_remote_gate_available(const Ranks &R)
{
    static const bool off = std::getenv("QSIM_NO_REMOTE_GATES") != nullptr;
    if (off) return false;
    if (R.size() > 1) return true;   // in-process rank group: every shard is addressable (peer access)
#ifndef QSIM_NO_NCCL
    Handle *h = R[0];
    if (h->world > 1 && h->comm) return ipc_setup(h) == 1;
#endif
    return false;
}

#ifndef QSIM_NO_NCCL
// Multi-process variant: which of its two allocations is each rank's current
// shard (one all-gather of a parity byte), the peer-memory kernel, then a
// stream-ordered barrier (1-element all-reduce) before anyone reuses a shard
// its partner may still be reading.
static int remote_gate_world(Handle *h, uint64_t cmask, uint64_t cvals, int q, const double2 U[4])
{
    if (int rc = flush_queue(h)) return rc;
    const int W = h->world, nl = h->nl;
    const int gb = h->pos[q] - nl;
    const int partner = h->rank ^ (1 << gb);
    uint64_t m = 0, v = 0;
    bool part = true;
    for (int c = 0; c < h->n && part; ++c) {
        if (!((cmask >> c) & 1)) continue;
        const int p = h->pos[c];
        const uint64_t want = (cvals >> c) & 1;
        if (p < nl) {
            m |= 1ull << p;
            v |= want << p;
        } else if ((((uint64_t)h->rank >> (p - nl)) & 1) != want) {
            part = false;
        }
    }
    unsigned char par = h->psi == h->own_buf[0] ? 0 : 1;
    std::vector<unsigned char> pars(W, 0);
    unsigned char *d = nullptr;
    if (cudaMalloc(&d, W + 1) != cudaSuccess) {
        cudaGetLastError();
        return fail(h, QSIM_ENOMEM, "remote gate buffer");
    }
    cudaMemcpyAsync(d, &par, 1, cudaMemcpyHostToDevice, h->stream);
    if (int rc = nccl_check(h, ncclAllGather(d, d + 1, 1, ncclUint8, h->comm, h->stream), "ncclAllGather")) return rc;
    cudaMemcpyAsync(pars.data(), d + 1, W, cudaMemcpyDeviceToHost, h->stream);
    cudaStreamSynchronize(h->stream);
    cudaFree(d);
    if (part) {
        const int b = (h->rank >> gb) & 1;
        const double2 *theirs = h->peer_buf[2 * partner + pars[partner]];
        launch_apply_2x2_remote(h, theirs, h->scratch, m, v, U[2 * b + b], U[2 * b + (1 - b)]);
    }
    // barrier: every rank's kernel has finished reading its partner's shard
    double *dz = nullptr;
    if (cudaMalloc(&dz, sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return fail(h, QSIM_ENOMEM, "remote gate barrier");
    }
    cudaMemsetAsync(dz, 0, sizeof(double), h->stream);
    int rc = nccl_check(h, ncclAllReduce(dz, dz, 1, ncclDouble, ncclSum, h->comm, h->stream), "barrier");
    cudaStreamSynchronize(h->stream);
    cudaFree(dz);
    if (rc) return rc;
    if (part) swap_buffers(h);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QSIM_OK : check_cuda(h, e, "remote gate");
}
#endif

// Every participating rank r computes its half of each pair from its own
// shard and its partner's (r ^ 2^(g-nl)) into its scratch shard; once both
// kernels of a pair are done (cross-stream events) the ranks swap shard and
// scratch.  No layout change, no staging copies.
// Multi-process world, rank-group passes: every rank's current shard mapped
// into this process (CUDA IPC, set up once; one all-gather of which of its two
// allocations each rank is using), and a stream-ordered barrier.
int dist_world_shards(Handle *h, std::vector<double2 *> &shards)
{
#ifndef QSIM_NO_NCCL
    if (h->world < 2 || !h->comm || ipc_setup(h) != 1) return 1;
    const int W = h->world;
    unsigned char par = h->psi == h->own_buf[0] ? 0 : 1;
    std::vector<unsigned char> pars(W, 0);
    unsigned char *d = nullptr;
    if (cudaMalloc(&d, W + 1) != cudaSuccess) {
        cudaGetLastError();
        return fail(h, QSIM_ENOMEM, "rank-group pass buffer");
    }
    cudaMemcpyAsync(d, &par, 1, cudaMemcpyHostToDevice, h->stream);
    int rc = nccl_check(h, ncclAllGather(d, d + 1, 1, ncclUint8, h->comm, h->stream), "ncclAllGather");
    cudaMemcpyAsync(pars.data(), d + 1, W, cudaMemcpyDeviceToHost, h->stream);
    cudaStreamSynchronize(h->stream);
    cudaFree(d);
    if (rc) return rc;
    shards.assign(W, nullptr);
    for (int r = 0; r < W; ++r) shards[r] = h->peer_buf[2 * r + pars[r]];
    return QSIM_OK;
#else
    (void)h;
    (void)shards;
    return 1;
#endif
}

int dist_world_barrier(Handle *h)
{
#ifndef QSIM_NO_NCCL
    double *dz = nullptr;
    if (cudaMalloc(&dz, sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return fail(h, QSIM_ENOMEM, "barrier buffer");
    }
    cudaMemsetAsync(dz, 0, sizeof(double), h->stream);
    int rc = nccl_check(h, ncclAllReduce(dz, dz, 1, ncclDouble, ncclSum, h->comm, h->stream), "barrier");
    cudaStreamSynchronize(h->stream);
    cudaFree(dz);
    return rc;
#else
    (void)h;
    return QSIM_OK;
#endif
}

int dist_remote_gate(const Ranks &R, uint64_t cmask, uint64_t cvals, int q, const double2 U[4])
{
#ifndef QSIM_NO_NCCL
    if (R.size() == 1) return remote_gate_world(R[0], cmask, cvals, q, U);
#endif
    if (int rc = flush_all(R)) return rc;
    const size_t P = R.size();
    const int nl = R[0]->nl;
    const int gb = R[0]->pos[q] - nl;
    std::vector<char> part(P, 0);
    std::vector<uint64_t> lm(P), lv(P);
    for (size_t r = 0; r < P; ++r) {
        Handle *h = R[r];
        uint64_t m = 0, v = 0;
        bool ok = true;
        for (int c = 0; c < h->n && ok; ++c) {
            if (!((cmask >> c) & 1)) continue;
            const int p = h->pos[c];
            const uint64_t want = (cvals >> c) & 1;
            if (p < nl) {
                m |= 1ull << p;
                v |= want << p;
            } else if ((((uint64_t)h->rank >> (p - nl)) & 1) != want) {
                ok = false;
            }
        }
        part[r] = ok;
        lm[r] = m;
        lv[r] = v;
        if (ok)
            if (int rc = ensure_scratch(h)) return rc;
    }
    std::vector<cudaEvent_t> pre(P), post(P);
    for (size_t r = 0; r < P; ++r) {
        cudaSetDevice(R[r]->device);
        cudaEventCreateWithFlags(&pre[r], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&post[r], cudaEventDisableTiming);
        cudaEventRecord(pre[r], R[r]->stream);
    }
    for (size_t r = 0; r < P; ++r) {
        if (!part[r]) continue;
        Handle *h = R[r];
        const size_t p = r ^ ((size_t)1 << gb);
        const int b = (h->rank >> gb) & 1;
        cudaSetDevice(h->device);
        cudaStreamWaitEvent(h->stream, pre[p], 0);   // the partner's shard is final
        launch_apply_2x2_remote(h, R[p]->psi, h->scratch, lm[r], lv[r], U[2 * b + b], U[2 * b + (1 - b)]);
        cudaEventRecord(post[r], h->stream);
    }
    for (size_t r = 0; r < P; ++r) {
        if (!part[r]) continue;
        const size_t p = r ^ ((size_t)1 << gb);
        cudaSetDevice(R[r]->device);
        cudaStreamWaitEvent(R[r]->stream, post[p], 0);   // the partner has read our shard
    }
    for (size_t r = 0; r < P; ++r) {
        if (part[r]) swap_buffers(R[r]);
        cudaSetDevice(R[r]->device);
        cudaEventDestroy(pre[r]);
        cudaEventDestroy(post[r]);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QSIM_OK : check_cuda(R[0], e, "remote gate");
}

int flush_all(const Ranks &R)
{
    for (Handle *h : R)
        if (int rc = flush_queue(h)) return rc;
    return QSIM_OK;
}

int dist_make_local(const Ranks &R, const std::vector<int> &need)
{
    Handle *h = R[0];
    if (h->world == 1) return QSIM_OK;
    bool all_local = true;
    for (int q : need) all_local &= h->pos[q] < h->nl;
    if (all_local) return QSIM_OK;
    if (int rc = flush_all(R)) return rc;
    std::vector<int> pos(h->pos, h->pos + h->n);
    std::vector<Step> steps;
    if (plan_make_local(h->n, h->nl, pos, need, steps)) return fail(h, QSIM_EINVAL, "too many qubits requested local");
    return run_steps(R, steps);
}

int dist_canonicalize(const Ranks &R)
{
    if (int rc = flush_all(R)) return rc;
    Handle *h0 = R[0];
    if (h0->world > 1) {
        std::vector<int> pos(h0->pos, h0->pos + h0->n);
        std::vector<Step> steps;
        if (plan_canonical_globals(h0->n, h0->nl, pos, steps)) return fail(h0, QSIM_EINVAL, "canonicalize plan");
        if (int rc = run_steps(R, steps)) return rc;
    }
    bool canon = true;
    for (int q = 0; q < h0->n; ++q) canon &= h0->pos[q] == h0->n - 1 - q;
    if (canon) return QSIM_OK;
    std::vector<int> perm(h0->nl);
    for (int q = 0; q < h0->n; ++q) {
        const int p = h0->pos[q];
        if (p < h0->nl) perm[p] = h0->n - 1 - q;
    }
    for (Handle *h : R) {
        permute_local(h, perm);
        for (int q = 0; q < h->n; ++q) h->pos[q] = h->n - 1 - q;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return check_cuda(h, e, "canonicalize");
        if (h->poisoned) return fail(h, QSIM_ECUDA, h->err);
    }
    return QSIM_OK;
}

int dist_sum_host(const Ranks &R, const std::vector<std::vector<double>> &parts, double *out, size_t count)
{
    Handle *h = R[0];
    if (R.size() > 1 || h->world == 1) {
        // all ranks are here: fixed rank order
        std::vector<double> acc(count, 0.0);
        for (size_t r = 0; r < R.size(); ++r)
            for (size_t i = 0; i < count; ++i) acc[i] += parts[r][i];
        std::memcpy(out, acc.data(), count * sizeof(double));
        return QSIM_OK;
    }
#ifndef QSIM_NO_NCCL
    // one rank of a multi-process world: allgather, then the same fixed-order sum
    double *d_in = nullptr, *d_out = nullptr;
    if (cudaMalloc(&d_in, count * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&d_out, count * h->world * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        if (d_in) cudaFree(d_in);
        return fail(h, QSIM_ENOMEM, "allgather buffers");
    }
    cudaMemcpyAsync(d_in, parts[0].data(), count * sizeof(double), cudaMemcpyHostToDevice, h->stream);
    int rc = nccl_check(h, ncclAllGather(d_in, d_out, count, ncclDouble, h->comm, h->stream), "ncclAllGather");
    std::vector<double> all(count * h->world);
    if (!rc) rc = check_cuda(h, cudaMemcpyAsync(all.data(), d_out, all.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "allgather copy");
    if (!rc) rc = check_cuda(h, cudaStreamSynchronize(h->stream), "allgather");
    cudaFree(d_in);
    cudaFree(d_out);
    if (rc) return rc;
    for (size_t i = 0; i < count; ++i) {
        double s = 0.0;
        for (int r = 0; r < h->world; ++r) s += all[(size_t)r * count + i];
        out[i] = s;
    }
    return QSIM_OK;
#else
    return fail(h, QSIM_ENCCL, "built without NCCL");
#endif
}

}  // namespace qs

// Exported planners for the host-side tests (no GPU needed).  Steps are
// written as triples (kind, a, b) into steps[0 .. 3*cap); returns the step
// count (or a negative QSIM_E* code); pos_io is updated in place.
extern "C" int qsim_plan_make_local(int n, int world, int *pos_io, const int *need, int nneed,
                                    int *steps, int cap)
{
    using namespace qs;
    int kg = 0;
    while ((1 << kg) < world) ++kg;
    std::vector<int> pos(pos_io, pos_io + n);
    std::vector<Step> st;
    if (int rc = plan_make_local(n, n - kg, pos, std::vector<int>(need, need + nneed), st)) return rc;
    for (int q = 0; q < n; ++q) pos_io[q] = pos[q];
    for (int i = 0; i < (int)st.size() && i < cap; ++i) {
        steps[3 * i] = st[i].kind; steps[3 * i + 1] = st[i].a; steps[3 * i + 2] = st[i].b;
    }
    return (int)st.size();
}

extern "C" int qsim_plan_canonical_globals(int n, int world, int *pos_io, int *steps, int cap)
{
    using namespace qs;
    int kg = 0;
    while ((1 << kg) < world) ++kg;
    std::vector<int> pos(pos_io, pos_io + n);
    std::vector<Step> st;
    if (int rc = plan_canonical_globals(n, n - kg, pos, st)) return rc;
    for (int q = 0; q < n; ++q) pos_io[q] = pos[q];
    for (int i = 0; i < (int)st.size() && i < cap; ++i) {
        steps[3 * i] = st[i].kind; steps[3 * i + 1] = st[i].a; steps[3 * i + 2] = st[i].b;
    }
    return (int)st.size();
}
