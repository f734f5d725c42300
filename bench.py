#!/usr/bin/env python3
"""Benchmark: BASELINE.json configs[2] (QFT on n = 28 qubits, complex128,
seeded complex-Gaussian input) through libqsim's C-ABI.

Metric (BASELINE.json): "state-vector GB/s per gate (% HBM peak) & circuit
time".  One step = the whole QFT circuit (28 H + 378 controlled R_d + 14
SWAP) on the 4 GiB state resident in HBM.  value = the
per-gate state-vector bandwidth in the paper's one-sweep-per-gate model: the
bytes each gate of the circuit must move when applied alone (dense/H:
2^(n+5) B, controlled R_d: 2^(n+3) B, SWAP: 2^(n+4) B; 1036 GiB at n = 28)
divided by the circuit time -- the unit says "effective" because fused passes
move far fewer bytes.  The bytes the passes really move and their fraction of
the measured HBM peak are in `roofline` (dominant kernel) and
config["hbm_gbs_achieved"] (whole circuit).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (one process per GPU;
the state is sharded on its top log2 N qubits, exchanges over NCCL).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_QUBITS = 28
SEED = 3
METRIC = "state-vector GB/s per gate (QFT circuit; % HBM peak in roofline) & circuit time"
UNIT = "GB/s effective (one-sweep-per-gate bytes / circuit time)"
WORKLOAD = "configs[2]: QFT circuit, n=28 complex128 (4 GiB), seeded complex-Gaussian input"


def gate_bytes(n):
    """Algorithmic bytes of the unfused QFT circuit (one sweep per gate)."""
    h = n * (1 << (n + 5))
    cr = (n * (n - 1) // 2) * (1 << (n + 3))
    sw = (n // 2) * (1 << (n + 4))
    return h + cr + sw, n + n * (n - 1) // 2 + n // 2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured", float(d.get("sm_max_mhz", 1965))
    return 6650.0, "fallback", 1965.0


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(n_full=N_QUBITS):
    """The oracle as it stands (plain C + OpenMP) on the host cores, on the
    bench's own configuration: the whole configs[2] QFT circuit at n = 28 on
    the same seeded Gaussian state (one run, ~25 s on 16 cores), timed around
    the circuit only; reported in the same per-gate unit."""
    import oracle as O
    psi = O.gaussian_state(n_full, SEED)
    t0 = time.perf_counter()
    O.qft(psi, 0, n_full, False)
    dt = time.perf_counter() - t0
    del psi
    gb, ng = gate_bytes(n_full)
    cores = O.get_threads()
    # one thread, the paper's 1-processor column, on a smaller sample
    n1 = 22
    psi1 = O.gaussian_state(n1, SEED)
    O.set_threads(1)
    t1 = time.perf_counter()
    O.qft(psi1, 0, n1, False)
    dt1 = time.perf_counter() - t1
    O.set_threads(0)
    gb1, ng1 = gate_bytes(n1)
    return {"value": gb / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"the full configs[2] circuit: oracle QFT on the n={n_full} seeded Gaussian state "
                      f"({ng} gates, one run, {dt:.1f} s)",
            "seconds": dt, "same_config": n_full == N_QUBITS,
            "single_thread": {"value": gb1 / dt1 / 1e9, "unit": UNIT, "cores": 1, "seconds": dt1,
                              "sample": f"oracle QFT circuit on n={n1} ({ng1} gates) on one host thread"}}


def qft_row_gates(n, j):
    """Row j of the QFT circuit: H(j), then R_{k-j}
    controlled by k on j for k > j; returns (kind, control, angle) tuples."""
    return [("h", -1, 0.0)] + [("r", k, math.pi / (1 << (k - j))) for k in range(j + 1, n)]


def run_reference(args):
    """The reference arm: the oracle on the host cores on our own config
    (configs[2], n = 28, the same seeded Gaussian state).  The whole circuit
    takes ~25 s, so each step is a bounded sample of it: one row of the QFT
    circuit (H(j) and its controlled R_d), rows taken in
    turn from j = 0; the per-gate unit makes rows comparable."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    import oracle as O
    n = args.ref_n
    psi = O.gaussian_state(n, SEED)
    Hm = np.array([[1, 1], [1, -1]], complex) / math.sqrt(2)
    times, gbs = [], []
    for i in range(args.warmup + args.steps):
        j = i % n
        gates = qft_row_gates(n, j)
        t0 = time.perf_counter()
        for kind, c, ang in gates:
            if kind == "h":
                O.apply_1q(psi, j, Hm)
            else:
                O.apply_ctrl(psi, 1 << c, 1 << c, j, np.diag([1.0, complex(math.cos(ang), math.sin(ang))]))
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            gbs.append(((1 << (n + 5)) + (len(gates) - 1) * (1 << (n + 3))) / 1e9)
    t = statistics.mean(times)
    value = sum(gbs) / sum(times)
    cores = O.get_threads()
    gb_full, ng_full = gate_bytes(N_QUBITS)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded complex Gaussian, DESIGN.md R19)",
        "config": {"workload": WORKLOAD, "n": N_QUBITS, "gates": ng_full, "gate_bytes": gb_full,
                   "state_bytes": 16 << N_QUBITS, "parallelism": "cpu-oracle",
                   "sample": f"each step: one row of the QFT circuit (H(j) + its controlled R_d) on the n={n} "
                             f"seeded Gaussian state, rows j = 0, 1, ... in turn, by the CPU oracle "
                             f"(plain C + OpenMP)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"oracle QFT-circuit rows at n={n}, {args.steps} timed steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cfg4_gate_bytes(n, layers=20):
    """Per-gate model of configs[4]: a Haar gate 2^(n+5) B, a noisy CNOT (a
    controlled dense 2x2, one control) 2^(n+4) B."""
    cnots = sum(len(range(l & 1, n - 1, 2)) for l in range(layers))
    return layers * n * (1 << (n + 5)) + cnots * (1 << (n + 4)), layers * n + cnots


def run_config4(args):
    """configs[4] (BASELINE.json): the noisy Haar + CNOT brickwork, n = 32,
    20 layers, sigma = 1e-3, p = 1e-4, seed 5, on one GPU; one step = the
    whole circuit from |0...0> (qsim_set_basis) to the read-out of the norm.
    The gate-list passes are FP64-bound, so the roofline object is the FP64
    pipe of the dominant kernel: algorithmic FP64 instructions per launch
    (16 per amplitude pair of a dense 2x2, the library's count) over its launch
    time, against 148 SMs x 64 FP64 FMA/clk x the max SM clock."""
    import torch
    from paper_quant_ph_0201042_b200 import qsim as Q
    from paper_quant_ph_0201042_b200 import workloads as W
    n = args.n if args.n != N_QUBITS else 32
    layers = 20
    torch.cuda.set_device(0)
    h = Q.qsim_create(n)
    stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
    events = []

    def step():
        # the whole circuit, executed: gates still queued at the end (the last
        # layer's) would otherwise be dropped by the next step's qsim_set_basis
        nonlocal events
        events = W.run_cfg4(h, n=n, layers=layers, seed=5, sigma=1e-3, p=1e-4)
        Q.qsim_sync(h)

    for _ in range(args.warmup):
        step()
    Q.qsim_sync(h)
    sampler = ClockSampler(0)
    sampler.start()
    time.sleep(0.3)
    l0 = Q.qsim_launch_count(h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    Q.qsim_sync(h)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = Q.qsim_launch_count(h) - l0
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    # end to end: the same step with its result (the norm and the event list) read back
    t0 = time.perf_counter()
    for _ in range(2):
        step()
        nrm = Q.qsim_norm(h)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / 2
    Q.qsim_profile(h, True)
    step()
    prof = Q.qsim_profile_json(h)
    prof.pop("_launches", None)
    Q.qsim_profile(h, False)
    gb, ngates = cfg4_gate_bytes(n, layers)
    value = gb / (ms * 1e-3) / 1e9
    peak_hbm, peak_kind, sm_max = load_peaks()
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    fp64_peak = 148 * 64 * sm_max * 1e6          # FP64 FMA-class instructions per second (lanes)
    ach = dom["fp64"] / (dom["ms"] * 1e-3)
    roof = {"bound": "fp64", "kernel": dom_name, "achieved": ach / 1e12, "peak": fp64_peak / 1e12,
            "unit": "T FP64 instr/s", "frac": ach / fp64_peak, "traffic": None,
            "peak_source": "148 SMs x 64 FP64 FMA/clk x sm_max_mhz (B200_PROFILING.md units; tools/microbench.cu "
                           "measured 58.4/clk/SM)",
            "fp64_per_launch": dom["fp64"] / dom["launches"], "ms_per_launch": dom["ms"] / dom["launches"],
            "launches_per_step": dom["launches"], "share_of_step": dom["ms"] / ms,
            "hbm_gbs_of_kernel": dom["bytes"] / (dom["ms"] * 1e-3) / 1e9}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Haar + noisy-CNOT brickwork, DESIGN.md R18)",
        "config": {"workload": f"configs[4]: noisy random circuit n={n}, 20 layers, sigma=1e-3, p=1e-4, seed 5",
                   "n": n, "gates": ngates, "gate_bytes": gb, "state_bytes": 16 << n, "parallelism": "sv-shard1",
                   "l2": f"inputs larger than L2 ({16 << n >> 30} GiB state)", "circuit_ms": ms,
                   "events_last_step": len(events), "norm_after": nrm},
        "roofline": roof,
        "cpu_baseline": None,
        "e2e": {"value": gb / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms, "h2d_bytes_per_step":
                ngates * 64, "d2h_bytes_per_step": 8 + 24 * len(events),
                "how": "run_cfg4 (gate matrices to the device as call parameters) + qsim_norm read-back"},
        "gpu_launches": launches, "clocks": clocks,
        "kernels": prof,
    }
    print(json.dumps(line), flush=True)
    Q.qsim_destroy(h)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_QUBITS)
    ap.add_argument("--ref-n", type=int, default=N_QUBITS)
    ap.add_argument("--cpu-n", type=int, default=N_QUBITS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=24)
    ap.add_argument("--profile-only", action="store_true", help="warm-up + steps only (for ncu)")
    ap.add_argument("--config", type=int, default=2, choices=[2, 4],
                    help="2: the headline QFT (default); 4: the noisy brickwork, FP64 roofline (one GPU)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 4:
        return run_config4(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus or world == 1, "launch with torchrun for --gpus > 1"
    if world > 1:
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)

    from paper_quant_ph_0201042_b200 import qsim as Q
    from paper_quant_ph_0201042_b200 import workloads as W

    n = args.n
    # --gpus N without torchrun: one process drives N ranks (qsim_create(n, N),
    # the in-process rank group; ranks share devices when fewer are visible)
    group = world == 1 and args.gpus > 1
    ranks = args.gpus if group else world
    if world > 1:
        uid = [Q.qsim_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        h = Q.qsim_create_dist(n, world, rank, local, uid[0])
    else:
        h = Q.qsim_create(n, ranks)
    stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        Q.qsim_qft(h, 0, n, False)

    Q.qsim_init_gaussian(h, SEED)
    for _ in range(args.warmup):
        step()
    Q.qsim_sync(h)
    if args.profile_only:
        for _ in range(args.steps):
            step()
        Q.qsim_sync(h)
        Q.qsim_destroy(h)
        return 0

    # ---------------- timed region (device time, CUDA events on the library's
    # stream; the library's per-launch profiler is off here so nothing sits
    # between the kernels)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    l0 = Q.qsim_launch_count(h)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = Q.qsim_launch_count(h) - l0
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # ---------------- the same steps again with the per-launch profiler on
    # (CUDA events around every launch on the library's stream): the
    # dominant kernel's launch durations for the roofline object
    Q.qsim_profile(h, True)
    for _ in range(args.steps):
        step()
    prof = Q.qsim_profile_json(h)
    per_launch = prof.pop("_launches", [])
    Q.qsim_profile(h, False)
    norm = Q.qsim_norm(h)

    gb, ngates = gate_bytes(n)
    value = gb / (ms * 1e-3) / 1e9      # whole-job GB/s (the state spans all ranks)
    peak, peak_kind, _ = load_peaks()

    # dominant kernel roofline (algorithmic bytes per launch / mean launch time)
    is_comm = lambda k: k.startswith("nccl_") or k.startswith("group_")
    ours = {k: v for k, v in prof.items() if not is_comm(k)}
    # the whole circuit's real HBM traffic: the algorithmic bytes of every launch
    pass_bytes = sum(v["bytes"] for v in ours.values()) / args.steps
    hbm_ach = pass_bytes / (ms * 1e-3) / 1e9   # per GPU: the profile covers rank 0 (its shard)
    passes = sum(v["launches"] for k, v in ours.items() if k.startswith("k_qft")) / args.steps
    comm = {k: v for k, v in prof.items() if is_comm(k)}
    dom = max(ours.items(), key=lambda kv: kv[1]["ms"]) if ours else None
    roof = None
    if dom:
        name, d = dom
        per_launch_ms = d["ms"] / d["launches"]
        bytes_per_launch = d["bytes"] / d["launches"]
        achieved = bytes_per_launch / (per_launch_ms * 1e-3) / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get(name)
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": f"{peak_kind} hbm_gbs",
                "bytes_per_launch": bytes_per_launch, "ms_per_launch": per_launch_ms,
                "launches_per_step": d["launches"] / args.steps,
                "share_of_step": d["ms"] / (ms * args.steps)}

    # NVLink: shard exchanges of the sharded QFT (rank 0's view; bytes = sent +
    # received, so per direction = half) against the measured 770 GB/s per
    # direction per GPU (B200_PROFILING.md; 900 nominal)
    nvlink = None
    if comm:
        cb = sum(v["bytes"] for v in comm.values())
        cms = sum(v["ms"] for v in comm.values())
        if cms > 0:
            ach = cb / 2 / (cms * 1e-3) / 1e9
            shared = group and torch.cuda.device_count() < ranks
            nvlink = {"bound": "nvlink", "achieved": ach, "peak": 770.0, "unit": "GB/s per direction",
                      "note": ("ranks share one device: device-local copies, not NVLink" if shared else
                               "rank 0's exchanges"),
                      "frac": ach / 770.0, "peak_source": "B200_PROFILING.md measured peer copy (900 nominal)",
                      "bytes_per_step": cb / args.steps, "ms_per_step": cms / args.steps,
                      "share_of_step": cms / (ms * args.steps),
                      "ops": {k: v["launches"] for k, v in comm.items()}}

    # ---------------- end to end: host buffers through the C-ABI.  Single GPU:
    # qsim_qft_host_stream pipelines the steps (copy in of step i+1 and copy
    # out of step i-1 overlap the transform of step i); every step still moves
    # its whole input in and its whole result out over PCIe inside the timed call.
    shard = 1 << (n - (world.bit_length() - 1))   # this process's slice (the whole state for a group)
    host_in = torch.empty(shard, dtype=torch.complex128, pin_memory=True).numpy()
    host_out = torch.empty(shard, dtype=torch.complex128, pin_memory=True).numpy()
    Q.qsim_get_state(h, rank * shard, shard, host_in)
    barrier()
    torch.cuda.synchronize()
    if world == 1 and not group:
        Q.qsim_qft_host_stream(h, 0, n, False, host_in, host_out, 1, 0, 0)   # warm the stages
        t0 = time.perf_counter()
        Q.qsim_qft_host_stream(h, 0, n, False, host_in, host_out, args.e2e_steps, 0, 0)
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        e2e_how = "qsim_qft_host_stream (pipelined host->device, transform, device->host)"
    else:
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            Q.qsim_set_state(h, rank * shard, host_in)
            step()
            Q.qsim_get_state(h, rank * shard, shard, host_out)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        e2e_how = "qsim_set_state + qsim_qft + qsim_get_state per step (serial)"
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": gb / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": shard * 16 * world, "d2h_bytes_per_step": shard * 16 * world,
           "how": e2e_how, "steps": args.e2e_steps}

    cpu = None
    if rank == 0 and world == 1 and not group and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_n)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": UNIT, "n_gpus": ranks, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded complex Gaussian, DESIGN.md R19)",
            "config": {"workload": WORKLOAD, "n": n, "gates": ngates, "gate_bytes": gb,
                       "state_bytes": 16 << n,
                       "parallelism": (f"sv-shard{ranks} (one process, rank group over "
                                       f"{torch.cuda.device_count()} visible device(s))" if group
                                       else f"sv-shard{world}"),
                       "l2": "inputs larger than L2 (4 GiB state vs 126 MB L2)",
                       "circuit_ms": ms, "effective_frac_of_hbm_peak": value / peak,
                       "hbm_gbs_achieved": hbm_ach, "hbm_frac_achieved": hbm_ach / peak,
                       "passes_per_step": passes, "norm_after": norm},
            "roofline": roof,
            "nvlink": nvlink,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "kernels": prof,
            "step_launches_ms": [round(x[1], 4) for x in per_launch[: len(per_launch) // max(args.steps, 1)]],
        }
        print(json.dumps(line), flush=True)
    Q.qsim_destroy(h)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
