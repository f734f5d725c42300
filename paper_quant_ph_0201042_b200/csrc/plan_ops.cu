// plan_ops.cu -- the gate queue's planner: queued gates -> fused tile passes
// (k_ops.cu / k_tma.cu k_ops_tma).
//
// Each pass reads and writes every amplitude once (one HBM sweep, the cost
// the paper pays per gate) and applies a whole run of
// gates in between.  Three steps per flush:
//
//  1. Pass selection (greedy, order-preserving up to commutation): a pass
//     collects, in queue order, every gate whose non-diagonal target is (or
//     can still become) one of its <= amax "active" positions; a gate that
//     cannot join blocks all of its positions for the rest of the scan.
//  2. Segment scheduling inside a pass.  A thread holds 16 amplitudes = a
//     4-bit register "window" of the tile; changing the window costs a
//     shared-memory transpose of the whole tile (as much time as ~2 dense
//     gates), so the planner orders the pass's gates -- any topological
//     order of their commutation DAG is the same operator -- to apply as
//     many gates per window as possible: for each candidate window (4-subsets
//     of the next dense targets) it simulates the closure of gates that
//     become applicable and keeps the best.
//  3. Merging: gates on one target that are adjacent in that order (up to
//     commutation) and are uncontrolled or controlled by the same window
//     qubit are multiplied into one 2x2 (or a pair of 2x2 selected by the
//     control, DENSE2): e.g. a Haar gate followed by a noisy CNOT on the same
//     target costs one register update instead of two.
//
// Two gates commute when every position they share is acted on diagonally
// by both (controls are diagonal projectors): exact, no numerical test.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <string>
#include <vector>

#include <cmath>

#include "qsim_internal.h"

namespace qs {

namespace {

// A gate of one pass in pass-local form.
struct POp {
    int dense;              // non-diagonal on tpos
    int tpos;               // target local position; -1: constant phase u[3]
    uint64_t cmask, cval;   // controls (local positions)
    int cs;                 // choice form: position selecting m1 (m0 where it is 0); -1: none
    double2 m0[4], m1[4];   // m1 == m0 when cs < 0
    uint64_t nmask, dmask;  // positions acted on non-diagonally / diagonally
    const double2 *tab;     // batched handle: per-trajectory matrices (merged on the device only)
    bool tab_own;           // tab is a product table this flush allocated (updated in place)
    bool dead;
};

inline bool conflict(const POp &a, const POp &b)
{
    return (a.nmask & (b.nmask | b.dmask)) || (b.nmask & (a.nmask | a.dmask));
}

inline bool eq(double2 a, double re, double im) { return a.x == re && a.y == im; }
inline bool is_ident(const double2 m[4]) { return eq(m[0], 1, 0) && eq(m[1], 0, 0) && eq(m[2], 0, 0) && eq(m[3], 1, 0); }
inline bool is_diagm(const double2 m[4]) { return eq(m[1], 0, 0) && eq(m[2], 0, 0); }

// C = A B (row-major 2x2 complex)
void mul2(const double2 A[4], const double2 B[4], double2 C[4])
{
    double2 r[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            const double2 a0 = A[2 * i], a1 = A[2 * i + 1], b0 = B[j], b1 = B[2 + j];
            r[2 * i + j] = make_double2(a0.x * b0.x - a0.y * b0.y + a1.x * b1.x - a1.y * b1.y,
                                        a0.x * b0.y + a0.y * b0.x + a1.x * b1.y + a1.y * b1.x);
        }
    std::memcpy(C, r, sizeof r);
}

void set_masks(POp &p)
{
    p.nmask = p.dense ? 1ull << p.tpos : 0;
    p.dmask = p.cmask | (p.cs >= 0 ? 1ull << p.cs : 0) | (!p.dense && p.tpos >= 0 ? 1ull << p.tpos : 0);
}

POp from_queue(const QOp &q)
{
    POp p;
    std::memset(&p, 0, sizeof p);
    p.dense = !q.diag || q.tab;
    p.tab = q.tab;
    p.tpos = q.tpos;
    p.cmask = q.cmask;
    p.cval = q.cval;
    p.cs = -1;
    for (int k = 0; k < 4; ++k) p.m0[k] = p.m1[k] = q.u[k];
    set_masks(p);
    return p;
}

struct Segment {
    int win[kOpsRegBits];      // tile bits held in registers
    std::vector<int> ops;   // op indices in application order
};

// Choice form (cs, m0, m1) of an op with at most one control (any local
// position: window, thread part or tile id); false if it has more.
bool choice_form(const POp &p, const std::vector<char> &in_win, int &cs, double2 m0[4], double2 m1[4])
{
    static const double2 I[4] = {{1, 0}, {0, 0}, {0, 0}, {1, 0}};
    if (p.cs >= 0) {
        if (p.cmask) return false;
        cs = p.cs;
        std::memcpy(m0, p.m0, 4 * sizeof(double2));
        std::memcpy(m1, p.m1, 4 * sizeof(double2));
        return true;
    }
    if (!p.cmask) {
        cs = -1;
        std::memcpy(m0, p.m0, 4 * sizeof(double2));
        std::memcpy(m1, p.m0, 4 * sizeof(double2));
        return true;
    }
    if (__builtin_popcountll(p.cmask) != 1) return false;
    const int c = __builtin_ctzll(p.cmask);
    cs = c;
    const bool v = (p.cval >> c) & 1;
    std::memcpy(v ? m1 : m0, p.m0, 4 * sizeof(double2));
    std::memcpy(v ? m0 : m1, I, 4 * sizeof(double2));
    return true;
}

// Merge B (applied after A, commuting with everything in between) into A.
bool try_merge(POp &A, const POp &B, const std::vector<char> &in_win)
{
    if (A.tpos < 0 || A.tpos != B.tpos || !in_win[A.tpos] || A.tab || B.tab) return false;
    int ca, cb;
    double2 a0[4], a1[4], b0[4], b1[4];
    if (!choice_form(A, in_win, ca, a0, a1) || !choice_form(B, in_win, cb, b0, b1)) return false;
    if (ca >= 0 && cb >= 0 && ca != cb) return false;
    if (!A.dense && !B.dense && (ca >= 0 || cb >= 0)) return false;   // keep cheap controlled phases
    const int cs = ca >= 0 ? ca : cb;
    double2 r0[4], r1[4];
    mul2(b0, a0, r0);
    mul2(b1, a1, r1);
    A.cmask = A.cval = 0;
    A.cs = cs;
    std::memcpy(A.m0, r0, sizeof r0);
    std::memcpy(A.m1, r1, sizeof r1);
    A.dense = !(is_diagm(r0) && is_diagm(r1));
    if (cs < 0 && !A.dense) A.cs = -1;
    set_masks(A);
    return true;
}

// Merge B into A when either carries per-trajectory matrices (batched
// handle): both uncontrolled on the same qubit; the product table B_t A_t is
// formed on the device into the handle's table arena (stream order puts it
// after the tables' producers and before the pass).  A run of k noisy gates
// or Pauli events on one qubit becomes one table lookup per tile.
bool try_merge_tab(Handle *h, POp &A, const POp &B)
{
    static const bool off = getenv("QSIM_NO_TAB_MERGE") != nullptr;
    if (off || A.tpos < 0 || A.tpos != B.tpos || A.cmask || B.cmask || A.cs >= 0 || B.cs >= 0) return false;
    if (!A.tab && !B.tab) return false;
    if (!A.dense || !B.dense) return false;
    const uint64_t count = 1ull << h->batch_b;
    const size_t need = 4 * count;
    double2 *out;
    if (A.tab_own) {
        out = const_cast<double2 *>(A.tab);   // a chain keeps one product table (element-wise in place)
    } else {
        if (!h->d_tabs || h->tabs_used + need > h->tabs_cap) return false;
        out = h->d_tabs + h->tabs_used;
        h->tabs_used += need;
    }
    launch_batch_mul(h, out, A.tab, A.m0, B.tab, B.m0, count);
    A.tab = out;
    A.tab_own = true;
    set_masks(A);
    return true;
}

// Order the ops of one pass into register-window segments (see header).
std::vector<Segment> schedule(const std::vector<POp> &ops, int nl, const std::vector<int> &tbit_of,
                              const std::vector<int> &tile)
{
    const int n = (int)ops.size();
    const int tbits = (int)tile.size();
    std::vector<std::vector<int>> succ(n);
    std::vector<int> npred(n, 0);
    {
        std::vector<int> lastN(nl, -1);
        std::vector<std::vector<int>> sinceD(nl);
        std::vector<int> pr;
        for (int j = 0; j < n; ++j) {
            pr.clear();
            const uint64_t dn = ops[j].dmask & ~ops[j].nmask;
            for (int p = 0; p < nl; ++p) {
                if ((ops[j].nmask >> p) & 1) {
                    if (lastN[p] >= 0) pr.push_back(lastN[p]);
                    pr.insert(pr.end(), sinceD[p].begin(), sinceD[p].end());
                } else if ((dn >> p) & 1) {
                    if (lastN[p] >= 0) pr.push_back(lastN[p]);
                }
            }
            std::sort(pr.begin(), pr.end());
            pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
            for (int i : pr) {
                succ[i].push_back(j);
                ++npred[j];
            }
            for (int p = 0; p < nl; ++p) {
                if ((ops[j].nmask >> p) & 1) {
                    lastN[p] = j;
                    sinceD[p].clear();
                } else if ((dn >> p) & 1) {
                    sinceD[p].push_back(j);
                }
            }
        }
    }
    std::vector<int> cnt = npred;
    std::vector<char> done(n, 0);
    int ndone = 0;
    std::vector<Segment> segs;
    std::vector<int> prev;
    for (int b = tbits - kOpsRegBits; b < tbits; ++b) prev.push_back(b);

    // closure of window W from the current state; commit = apply it
    std::vector<int> c2;
    std::vector<int> taken;
    auto closure = [&](const std::vector<int> &W, bool commit) -> int {
        uint32_t wmask = 0;
        for (int b : W) wmask |= 1u << b;
        c2 = cnt;
        taken.clear();
        std::priority_queue<int, std::vector<int>, std::greater<int>> pq;
        for (int j = 0; j < n; ++j)
            if (!done[j] && c2[j] == 0) pq.push(j);
        int score = 0;
        std::vector<int> skipped;
        while (!pq.empty()) {
            const int j = pq.top();
            pq.pop();
            const POp &o = ops[j];
            if (o.dense && !((wmask >> tbit_of[o.tpos]) & 1)) continue;   // stays for a later window
            taken.push_back(j);
            if (o.dense) {
                score += 4;
                bool cw = true;
                for (int p = 0; p < nl; ++p)
                    if (((o.cmask >> p) & 1) && tbit_of[p] >= 0 && !((wmask >> tbit_of[p]) & 1)) cw = false;
                score += cw;
            }
            for (int s : succ[j])
                if (--c2[s] == 0) pq.push(s);
        }
        if (commit) {
            for (int j : taken) {
                done[j] = 1;
                ++ndone;
            }
            cnt = c2;
        }
        return score;
    };

    while (ndone < n) {
        std::vector<int> cand;
        for (int j = 0; j < n && (int)cand.size() < 2 * kOpsRegBits; ++j) {
            if (done[j] || !ops[j].dense) continue;
            const int t = tbit_of[ops[j].tpos];
            if (std::find(cand.begin(), cand.end(), t) == cand.end()) cand.push_back(t);
        }
        std::vector<int> best;
        if ((int)cand.size() <= kOpsRegBits) {
            best = cand;
            for (int b : prev)
                if ((int)best.size() < kOpsRegBits && std::find(best.begin(), best.end(), b) == best.end()) best.push_back(b);
            // filler: highest tile positions first (low positions stay lane bits)
            std::vector<int> byp(tbits);
            for (int b = 0; b < tbits; ++b) byp[b] = b;
            std::sort(byp.begin(), byp.end(), [&](int x, int y) { return tile[x] > tile[y]; });
            for (int b : byp)
                if ((int)best.size() < kOpsRegBits && std::find(best.begin(), best.end(), b) == best.end()) best.push_back(b);
        } else {
            // every kOpsRegBits-subset of the candidates (<= C(10, 5) = 252)
            int bscore = -1;
            const int m = (int)cand.size();
            std::vector<int> idx(kOpsRegBits);
            for (int k = 0; k < kOpsRegBits; ++k) idx[k] = k;
            while (true) {
                std::vector<int> W(kOpsRegBits);
                for (int k = 0; k < kOpsRegBits; ++k) W[k] = cand[idx[k]];
                const int sc = closure(W, false);
                if (sc > bscore) {
                    bscore = sc;
                    best = W;
                }
                int k = kOpsRegBits - 1;
                while (k >= 0 && idx[k] == m - kOpsRegBits + k) --k;
                if (k < 0) break;
                ++idx[k];
                for (int l = k + 1; l < kOpsRegBits; ++l) idx[l] = idx[l - 1] + 1;
            }
        }
        std::sort(best.begin(), best.end());
        closure(best, true);
        Segment sg;
        for (int b = 0; b < kOpsRegBits; ++b) sg.win[b] = best[b];
        sg.ops = taken;
        segs.push_back(sg);
        prev = best;
    }
    return segs;
}

// The interpreter's dispatch word of an encoded op (qsim_internal.h OPC_*):
// one case id for (kind, window bits, window controls) plus the run-time
// checks the op needs, so the device takes one indexed branch per op.
uint32_t op_code(const GOp &g)
{
    uint32_t c = OPC_OTHER;
    const uint32_t wc = g.wm != 0;
    switch (g.kind) {
    case GOP_DENSE: c = OPC_DENSE + g.rb + 5 * wc; break;
    case GOP_DENSET: c = (OPC_DENSE + g.rb + 5 * wc) | kOpTraj; break;
    case GOP_CDENSE: c = OPC_CDENSE + g.rb * 10 + g.cs * 2 + g.cv; break;
    case GOP_DENSE2: c = OPC_DENSE2 + g.rb * 5 + g.cs; break;
    case GOP_DIAGW: c = OPC_DIAGW + g.rb * 4 + 2 * wc + (g.u[0].x == 1.0 && g.u[0].y == 0.0); break;
    default: break;
    }
    if (g.fm) c |= kOpChkFixed;
    if (g.tm) c |= kOpChkThread;
    if (g.kind == GOP_DENSE && (g.tsel != 0 || g.fsel != 0xff)) c |= kOpSel;
    return c;
}

bool plan_log()
{
    static const bool on = std::getenv("QSIM_PLAN_LOG") != nullptr;
    return on;
}

int launch_check(Handle *h, const char *what)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return check_cuda(h, e, what);
    if (h->poisoned) return fail(h, QSIM_ECUDA, h->err);
    return QSIM_OK;
}

}  // namespace

int flush_queue(Handle *h)
{
    cudaSetDevice(h->device);   // members of a rank group may live on different devices
    if (h->queue.empty()) {
        h->tabs_used = 0;
        return QSIM_OK;
    }
    std::vector<QOp> rem;
    rem.swap(h->queue);
    const int nl = h->nl;
    // batched handle: trajectory-index positions are never tile bits (a tile
    // belongs to one trajectory, whose matrices DENSET ops look up)
    std::vector<char> is_batch(nl, 0);
    int nbl = 0;
    for (int q = 0; q < h->batch_b; ++q)
        if (h->pos[q] < nl) {
            is_batch[h->pos[q]] = 1;
            ++nbl;
        }
    const int nreg = nl - nbl;
    const int tbits = std::min(kTileMaxBits, nreg);
    static const int npassive = std::getenv("QSIM_OPS_PASSIVE") ? std::atoi(std::getenv("QSIM_OPS_PASSIVE")) : 3;
    const int amax = nreg <= kTileMaxBits ? nreg : kTileMaxBits - npassive;
    constexpr size_t kPassCap = 512;   // bounds the planner's work per pass
    static thread_local OpsLaunch L;   // 28 KiB, copied into the launch parameters
    while (!rem.empty()) {
        // ---- 1. pass selection: the closure of the queue (in order, up to
        // commutation: a gate that cannot join blocks its positions) under an
        // active set built greedily, or under each window of amax consecutive
        // positions; the candidate applying the most register work wins.  A
        // window keeps a brickwork's light cone together (the greedy set
        // drifts into every other qubit, one layer per pass) and makes the
        // tile a TMA box.
        struct Sel {
            std::vector<char> take;
            std::vector<int> act;
            double w = 0.0;
        };
        auto closure = [&](uint64_t allowed) {   // allowed: active-position mask (~0: any)
            Sel s;
            s.take.assign(rem.size(), 0);
            uint64_t is_act = 0, blocked = 0;
            size_t ntake = 0;
            for (size_t i = 0; i < rem.size(); ++i) {
                const QOp &op = rem[i];
                uint64_t touch = op.cmask;
                if (op.tpos >= 0) touch |= 1ull << op.tpos;
                bool ok = ntake < kPassCap && !(touch & blocked);
                if (ok && !op.diag && !((is_act >> op.tpos) & 1)) {
                    if ((int)s.act.size() < amax && ((allowed >> op.tpos) & 1)) {
                        s.act.push_back(op.tpos);
                        is_act |= 1ull << op.tpos;
                    } else {
                        ok = false;
                    }
                }
                if (ok) {
                    s.take[i] = 1;
                    ++ntake;
                    s.w += op.diag ? 0.5 : 1.0;
                } else {
                    blocked |= touch;
                }
            }
            return s;
        };
        static const bool greedy_only = std::getenv("QSIM_PASS_GREEDY") != nullptr;
        Sel best = closure(~0ull);
        if (!greedy_only && nl > amax) {
            uint64_t batch_mask = 0;
            for (int p = 0; p < nl; ++p)
                if (is_batch[p]) batch_mask |= 1ull << p;
            for (int p0 = 0; p0 + amax <= nl; ++p0) {
                const uint64_t win = (((1ull << amax) - 1) << p0) & ~batch_mask;
                Sel s = closure(win);
                // a window's tile is a TMA box (k_ops_pp, ~7% faster per pass):
                // it wins ties with the greedy set and a 5% margin
                if (s.w * 1.05 > best.w) best = std::move(s);
            }
        }
        std::vector<int> act = best.act;
        std::vector<QOp> take, left;
        for (size_t i = 0; i < rem.size(); ++i) (best.take[i] ? take : left).push_back(rem[i]);
        rem.swap(left);
        // A pass of one sparse gate (controlled, or a phase on half the
        // amplitudes) reads and writes every amplitude; the unfused kernel
        // touches only the amplitudes the gate changes.  Measured on B200
        // (ncu dram__bytes, profiles/r2_lowgates.md): DRAM reads move whole
        // 128-byte lines (8 amplitudes), writes 32-byte sectors (2), so with
        // the masked positions m the unfused kernel moves S 2^-|m >> 3| read +
        // S 2^-|m >> 1| written against the pass's 2 S -- it wins below ~1.6 S
        // (CR on positions (1,2): 1.08 vs 1.35 ms at n = 28; (2,3): 0.63 vs
        // 1.36; position 0 in the mask touches every line and half the sectors or
        // more: the pass, measured no slower).
        if (take.size() == 1 && !take[0].tab) {
            const QOp &q = take[0];
            uint64_t m = q.cmask;
            if (q.diag && q.tpos >= 0 && q.u[0].x == 1.0 && q.u[0].y == 0.0) m |= 1ull << q.tpos;
            if (q.diag && q.tpos < 0) m = q.cmask;
            const double traffic = std::ldexp(1.0, -__builtin_popcountll(m >> 3)) +
                                   std::ldexp(1.0, -__builtin_popcountll(m >> 1));
            if (m && !(m & 1) && traffic <= 1.6) {
                run_gate_unfused(h, q);
                if (int rc = launch_check(h, "gate")) return rc;
                continue;
            }
        }
        // tile: active + passive lowest positions
        std::vector<int> tile(act);
        std::vector<int> tbit_of(nl, -1);
        for (size_t b = 0; b < act.size(); ++b) tbit_of[act[b]] = (int)b;
        for (int p = 0; p < nl && (int)tile.size() < tbits; ++p)
            if (tbit_of[p] < 0 && !is_batch[p]) {
                tbit_of[p] = (int)tile.size();
                tile.push_back(p);
            }
        OpsPass &P = L.P;
        std::memset(&P, 0, sizeof P);
        P.tbits = tbits;
        for (int b = 0; b < tbits; ++b) P.in_pos[b] = tile[b];
        std::vector<int> fix_of(nl, -1);
        for (int p = 0; p < nl; ++p)
            if (tbit_of[p] < 0) {
                fix_of[p] = P.nfix;
                P.fin_pos[P.nfix++] = p;
            }
        for (int q = 0; q < h->batch_b; ++q) {
            const int p = h->pos[q];
            const int sh = h->batch_b - 1 - q;   // qubit 0 = MSB of the trajectory index
            if (p < nl) {
                P.bat_fix[P.nbat] = fix_of[p];
                P.bat_sh[P.nbat++] = sh;
            } else {
                P.bat_rank |= (uint32_t)(((uint64_t)h->rank >> (p - nl)) & 1u) << sh;
            }
        }

        // ---- 2. segments, 3. merging
        std::vector<POp> ops;
        ops.reserve(take.size());
        for (const QOp &q : take) ops.push_back(from_queue(q));
        std::vector<Segment> segs = schedule(ops, nl, tbit_of, tile);
        std::vector<std::vector<GOp>> enc(segs.size());
        for (size_t s = 0; s < segs.size(); ++s) {
            const Segment &sg = segs[s];
            std::vector<char> in_win(nl, 0);
            for (int b = 0; b < kOpsRegBits; ++b) in_win[tile[sg.win[b]]] = 1;
            const std::vector<int> &Ls = sg.ops;
            for (size_t jj = 0; jj < Ls.size(); ++jj) {
                POp &B = ops[Ls[jj]];
                for (size_t ii = jj; ii-- > 0;) {
                    POp &A = ops[Ls[ii]];
                    if (A.dead) continue;
                    if (A.tpos == B.tpos && (try_merge(A, B, in_win) || try_merge_tab(h, A, B))) {
                        B.dead = true;
                        break;
                    }
                    if (conflict(A, B)) break;
                }
            }
            auto win_idx = [&](int pos) {
                const int t = tbit_of[pos];
                for (int b = 0; b < kOpsRegBits; ++b)
                    if (sg.win[b] == t) return b;
                return -1;
            };
            for (int j : Ls) {
                const POp &q = ops[j];
                if (q.dead) continue;
                GOp g;
                std::memset(&g, 0, sizeof g);
                for (int k = 0; k < 4; ++k) {
                    g.u[k] = q.m0[k];
                    g.u[4 + k] = q.m1[k];
                }
                g.fsel = 0xff;
                if (q.tab) {
                    g.kind = GOP_DENSET;
                    g.rb = (uint8_t)win_idx(q.tpos);
                    g.tab = q.tab;
                }
                if (q.cs >= 0 && win_idx(q.cs) >= 0) {
                    // choice form (merged run) selected by a window bit: static slot selection
                    g.rb = (uint8_t)win_idx(q.tpos);
                    g.cs = (uint8_t)win_idx(q.cs);
                    if (is_ident(q.m0)) {
                        g.kind = GOP_CDENSE;
                        g.cv = 1;
                        for (int k = 0; k < 4; ++k) g.u[k] = q.m1[k];
                    } else if (is_ident(q.m1)) {
                        g.kind = GOP_CDENSE;
                        g.cv = 0;
                    } else {
                        g.kind = GOP_DENSE2;
                    }
                    enc[s].push_back(g);
                    continue;
                }
                if (q.cs >= 0) {
                    // choice by a thread-part bit (one matrix per thread) or a
                    // tile-id bit (one matrix per tile; a tile whose matrix is I skips)
                    g.kind = GOP_DENSE;
                    g.rb = (uint8_t)win_idx(q.tpos);
                    const int tb = tbit_of[q.cs];
                    if (tb >= 0) {
                        g.tsel = 1u << tb;
                    } else if (is_ident(q.m0) || is_ident(q.m1)) {
                        const bool one = is_ident(q.m0);
                        g.fm = 1ull << fix_of[q.cs];
                        g.fv = one ? g.fm : 0;
                        for (int k = 0; k < 4; ++k) g.u[k] = g.u[4 + k] = one ? q.m1[k] : q.m0[k];
                    } else {
                        g.fsel = (uint8_t)fix_of[q.cs];
                    }
                    enc[s].push_back(g);
                    continue;
                }
                if (q.tab) {
                    // DENSET set above; controls below
                } else if (q.dense) {
                    g.kind = GOP_DENSE;
                    g.rb = (uint8_t)win_idx(q.tpos);
                } else if (q.tpos < 0) {
                    g.kind = GOP_PHASE;
                } else if (tbit_of[q.tpos] >= 0 && win_idx(q.tpos) >= 0) {
                    g.kind = GOP_DIAGW;
                    g.rb = (uint8_t)win_idx(q.tpos);
                } else if (tbit_of[q.tpos] >= 0) {
                    g.kind = GOP_DIAGT;
                    g.tb = 1u << tbit_of[q.tpos];
                } else {
                    g.kind = GOP_DIAGF;
                    g.fbit = (uint32_t)fix_of[q.tpos];
                }
                for (int p = 0; p < nl; ++p) {
                    if (!((q.cmask >> p) & 1)) continue;
                    const uint64_t want = (q.cval >> p) & 1;
                    if (tbit_of[p] >= 0) {
                        const int w = win_idx(p);
                        if (w >= 0) {
                            g.wm |= (uint8_t)(1u << w);
                            g.wv |= (uint8_t)(want << w);
                        } else {
                            g.tm |= 1u << tbit_of[p];
                            g.tv |= (uint32_t)want << tbit_of[p];
                        }
                    } else {
                        g.fm |= 1ull << fix_of[p];
                        g.fv |= want << fix_of[p];
                    }
                }
                // a dense gate with exactly one control, on a window bit: static slot selection
                if (g.kind == GOP_DENSE && g.tm == 0 && g.fm == 0 && __builtin_popcount(g.wm) == 1) {
                    g.kind = GOP_CDENSE;
                    g.cs = (uint8_t)__builtin_ctz(g.wm);
                    g.cv = g.wv ? 1 : 0;
                    g.wm = g.wv = 0;
                }
                enc[s].push_back(g);
            }
        }
        // ---- launches: consecutive segments, <= kMaxSegs segments and <= kOpsParam ops each
        struct Piece { int seg; size_t b, e; };
        std::vector<Piece> pieces;
        for (size_t s = 0; s < segs.size(); ++s) {
            const size_t m = enc[s].size();
            for (size_t b = 0; b < m || (b == 0 && m == 0); b += kOpsParam) {
                pieces.push_back({(int)s, b, std::min(m, b + (size_t)kOpsParam)});
                if (m == 0) break;
            }
        }
        size_t pi = 0;
        while (pi < pieces.size()) {
            size_t pe = pi;
            size_t nops = 0;
            while (pe < pieces.size() && (int)(pe - pi) < kMaxSegs &&
                   nops + (pieces[pe].e - pieces[pe].b) <= (size_t)kOpsParam) {
                nops += pieces[pe].e - pieces[pe].b;
                ++pe;
            }
            P.nseg = (int)(pe - pi);
            P.nops = 0;
            for (size_t k = pi; k < pe; ++k) {
                const Segment &sg = segs[pieces[k].seg];
                OpsSeg &os = P.seg[k - pi];
                for (int b = 0; b < kOpsRegBits; ++b) os.win[b] = sg.win[b];
                std::vector<int> rest;
                for (int b = 0; b < tbits; ++b)
                    if (std::find(sg.win, sg.win + kOpsRegBits, b) == sg.win + kOpsRegBits) rest.push_back(b);
                // first/last segment of a launch: thread bits by position (coalesced gather/scatter)
                if (k == pi || k + 1 == pe)
                    std::stable_sort(rest.begin(), rest.end(), [&](int x, int y) { return tile[x] < tile[y]; });
                for (size_t t = 0; t < rest.size(); ++t) os.order[t] = rest[t];
                os.op_begin = P.nops;
                for (size_t i = pieces[k].b; i < pieces[k].e; ++i) {
                    GOp &g = L.ops[P.nops++];
                    g = enc[pieces[k].seg][i];
                    g.code = op_code(g);
                }
                os.op_end = P.nops;
            }
            if (plan_log()) {
                int cnt[8] = {0};
                int thr = 0;
                for (int i = 0; i < P.nops; ++i) {
                    ++cnt[L.ops[i].kind & 7];
                    thr += L.ops[i].tm != 0;
                }
                std::vector<int> tp(P.in_pos, P.in_pos + P.tbits);
                std::sort(tp.begin(), tp.end());
                std::string tps;
                for (int x : tp) tps += std::to_string(x) + ",";
                std::fprintf(stderr,
                             "[qsim plan] nl=%d tile=%d nseg=%d nops=%d dense=%d cdense=%d dense2=%d diagw=%d "
                             "diagt=%d diagf=%d phase=%d denset=%d thread-ctrl=%d positions=%s\n",
                             nl, tbits, P.nseg, P.nops, cnt[GOP_DENSE], cnt[GOP_CDENSE], cnt[GOP_DENSE2],
                             cnt[GOP_DIAGW], cnt[GOP_DIAGT], cnt[GOP_DIAGF], cnt[GOP_PHASE], cnt[GOP_DENSET], thr,
                             tps.c_str());
            }
            prof_set_fp64(h, ops_fp64(L));
            launch_ops_pass(h, L);
            if (int rc = launch_check(h, "fused gate pass")) return rc;
            pi = pe;
        }
    }
    h->tabs_used = 0;   // every queued table is consumed by the launches above (stream order)
    return QSIM_OK;
}

uint64_t ops_fp64(const OpsLaunch &L)
{
    const OpsPass &P = L.P;
    const double amps = std::ldexp(1.0, P.tbits + P.nfix);
    double per_amp = 0.0;
    for (int i = 0; i < P.nops; ++i) {
        const GOp &g = L.ops[i];
        double c;
        switch (g.kind) {
        case GOP_DENSE: case GOP_DENSE2: case GOP_DENSET: c = 8.0; break;
        case GOP_CDENSE: c = 4.0; break;
        case GOP_DIAGW: c = (g.u[0].x == 1.0 && g.u[0].y == 0.0) ? 2.0 : 4.0; break;
        default: c = 4.0; break;
        }
        c = std::ldexp(c, -__builtin_popcountll(g.fm) - __builtin_popcount(g.tm) - __builtin_popcount(g.wm));
        per_amp += c;
    }
    return (uint64_t)(per_amp * amps);
}

}  // namespace qs
