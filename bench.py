#!/usr/bin/env python
"""Benchmark of the TANQ hot path on B200 (contract: see DESIGN.md §Measurement).

One step = the whole hot path over the workload:
reset rho to |0..0><0..0|, execute the noise-bound, fused plan of the circuit (gate kernels +
global-qubit remaps), reduce the readout-noisy probabilities from the diagonal.

Default workload: BASELINE.json configs[3] -- 16-qubit QPE-style circuit with calibrated
device noise (68.7 GB density matrix), the largest configuration of the metric's n=14-18
range that fits one B200.  With --gpus N (torchrun, one process per GPU) the same state is
partitioned over N GPUs by its high qubit bits (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config C] [--n n]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused-gate updates/s & HBM GB/s vs 8 TB/s, n=14–18 qubit DM, 1/2/4/8 GPU"
UNIT = "fused-gate updates/s"
CONFIG_NAMES = {
    3: "config3: 14-qubit random layered depth 100, calibrated depol+thermal noise",
    4: "config4: 16-qubit QPE-style circuit, calibrated device noise (depol+thermal+readout)",
    5: "config5: 18-qubit VQE ansatz, calibrated noise + 69 Pauli expectations",
}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def fp64_tensor_peak():
    """FP64 tensor (DMMA.8x8x4) peak measured on this pool by microbench/ubench.cu
    (profiles/r01_microbench_b200.txt); MEASURED_PEAKS.json carries no FP64 figure."""
    import re
    p = os.path.join(ROOT, "profiles", "r01_microbench_b200.txt")
    if os.path.exists(p):
        vals = [float(x) for x in re.findall(r"DMMA m8n8k4.*?: ([0-9.]+) TFLOP/s", open(p).read())]
        if vals:
            return max(vals), "measured DMMA.8x8x4 microbench (profiles/r01_microbench_b200.txt)"
    return 37.2, "nominal 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"


def ncu_traffic(kernel: str, alg_bytes_per_launch: float):
    """dram read+write bytes per launch of `kernel`: the DRAM/algorithmic byte ratio of the
    committed ncu --set full capture (profiles/ncu_traffic.json) times this launch's bytes."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p)).get(kernel)
    if not isinstance(d, dict):
        return None, None
    return d["ratio"] * alg_bytes_per_launch, f"{d['source']} (n={d['n_qubits']}, ratio {d['ratio']:.4f})"


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------------------------------
# CPU baseline: the oracle as it stands, on a bounded sample of the same workload
# --------------------------------------------------------------------------------------
def plan_counts(config: int, n: int, world: int, fuse: int, kmax: int):
    """Fused-gate updates per circuit of the GPU plan, from the committed table written by
    scripts/plan_counts.py (the reference arm must not load libtanq.so to count them)."""
    p = os.path.join(ROOT, "workloads", "plan_counts.json")
    key = f"config{config}:n{n}:gpus{world}:fuse{fuse}:kmax{kmax}"
    d = json.load(open(p)) if os.path.exists(p) else {}
    if key not in d:
        raise SystemExit(f"no plan count for {key}: run scripts/plan_counts.py")
    return d[key]


def gate_classes(circ, nm):
    """Basis gates grouped by their oracle channel sequence (kind, arity, channel kinds)."""
    from oracle import channels
    out = {}
    for op in circ.ops:
        seq = channels.gate_channel_sequence(op, nm)
        key = (op.kind, len(op.qubits), tuple((k, len(q)) for k, q, _ in seq))
        out.setdefault(key, []).append(op)
    return out


def oracle_estimate(config: int, n_full: int, gate_updates: int, budget_s: float = 8.0,
                    n_sample: int = 13):
    """Oracle seconds per whole n_full circuit from a bounded, representative sample: every
    basis gate of the circuit belongs to one of a few channel-sequence classes (e.g. config 4:
    RZ = 1 Kraus channel; SX/X = U, AD, PD, 1q depolarizing; CX = U, 4 thermal, 2q
    depolarizing); one instance of each class is timed on the oracle at n_sample (<= n_full)
    qubits, repeated round-robin while the budget lasts, and the circuit time is
    sum_class count(class) x mean time(class) x 4^(n_full - n_sample) (the oracle's per-gate
    work is O(4^n): every block of the dense rho).  value = the GPU plan's fused-gate updates
    per circuit / that time."""
    import workloads as W
    from oracle import channels, dense

    n_s = min(n_full, n_sample)
    c_full, nm_full = W.config_workload(config, n=n_full)
    c_s, nm_s = W.config_workload(config, n=n_s)
    full_cls = gate_classes(c_full, nm_full)
    samp_cls = gate_classes(c_s, nm_s)
    missing = [k for k in full_cls if k not in samp_cls]
    if missing:
        raise RuntimeError(f"gate classes {missing} absent at n={n_s}")
    rho = dense.ground(n_s)
    dense.lib()
    first = next(iter(samp_cls.values()))[0]        # untimed: OpenMP pool + page warm-up
    dense.apply_channel_seq(rho, n_s, channels.gate_channel_sequence(first, nm_s))
    times = {k: [] for k in full_cls}
    t0 = time.perf_counter()
    while True:
        for k in full_cls:
            inst = samp_cls[k]           # instances spread over the circuit (golden-ratio stride)
            op = inst[int(len(times[k]) * 0.6180339887 * len(inst) + len(inst) // 2) % len(inst)]
            a = time.perf_counter()
            dense.apply_channel_seq(rho, n_s, channels.gate_channel_sequence(op, nm_s))
            times[k].append(time.perf_counter() - a)
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    del rho
    scale = 4.0 ** (n_full - n_s)
    per = {k: statistics.fmean(v) for k, v in times.items()}
    t_circuit = sum(len(full_cls[k]) * per[k] * scale for k in full_cls)
    desc = "; ".join(f"{k[0]}(k={k[1]}, {len(k[2])} channels) x{len(full_cls[k])}: "
                     f"{per[k] * 1e3:.0f} ms at n={n_s} ({len(times[k])} runs)" for k in full_cls)
    sample = (f"oracle (oracle/dense.c, OpenMP, all host cores) timed one instance of each of the "
              f"{len(full_cls)} channel-sequence classes of the config-{config} circuit on a dense "
              f"n={n_s} rho for {dt:.1f} s [{desc}]; circuit time = sum over the {len(c_full.ops)} "
              f"basis gates of the n={n_full} circuit of their class time x 4^({n_full}-{n_s}) = "
              f"{t_circuit:.0f} s; value = the GPU plan's {gate_updates} fused-gate updates per "
              f"circuit / that time")
    return {"value": gate_updates / t_circuit, "unit": UNIT, "cores": os.cpu_count(),
            "kind": "oracle", "sample": sample, "seconds": dt, "circuit_s_estimated": t_circuit}


def oracle_whole_circuit(config: int, n: int):
    """The whole config circuit at a small n, oracle end to end (no sampling, no scaling)."""
    import workloads as W
    from oracle import dense
    c, nm = W.config_workload(config, n=n)
    dense.lib()
    t0 = time.perf_counter()
    rho = dense.run(c, nm)
    p = dense.probs(rho, n, dense.readout_of(nm))
    dt = time.perf_counter() - t0
    return dt, p, c, nm


def workload_config(args, c, counts) -> dict:
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": CONFIG_NAMES.get(args.config, str(args.config)),
            "n_qubits": c.n, "gates": len(c.ops), "gate_updates": counts["gate_updates"],
            "fusion": f"fuse={args.fuse} k_max={args.kmax}", "state_bytes": 16 * 4 ** c.n,
            "l2": ("inputs larger than L2 (state >> 126 MB)" if 16 * 4 ** c.n > 5e8
                   else "state fits L2 (no flush)")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    import workloads as W
    c, nm = W.config_workload(args.config, n=args.n)
    counts = plan_counts(args.config, c.n, world, args.fuse, args.kmax)
    for _ in range(args.warmup):
        oracle_estimate(args.config, c.n, counts["gate_updates"], budget_s=args.ref_budget / 4)
    vals = []
    t0 = time.perf_counter()
    cb = None
    for _ in range(args.steps):
        cb = oracle_estimate(args.config, c.n, counts["gate_updates"], budget_s=args.ref_budget)
        vals.append(cb["value"])
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, c, counts),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb["cores"],
                             "kind": "oracle", "sample": cb["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def build_nccl_shim() -> str:
    """tests/nccl_shim: host-staged stand-in for the NCCL calls libtanq makes, for running N
    ranks on fewer GPUs (a functional check of the N > 1 path, never a multi-GPU timing)."""
    out = os.path.join("/tmp", f"tanq_nccl_shim_{os.getuid()}.so")
    src = os.path.join(ROOT, "tests", "nccl_shim", "nccl_shim.cpp")
    subprocess.check_call(["g++", "-O2", "-shared", "-fPIC", "-std=c++17",
                           "-I/usr/local/cuda/include", src, "-o", out,
                           "-L/usr/local/cuda/lib64", "-lcudart", "-lpthread"])
    return out


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without torchrun: start the N ranks here (one process per GPU,
    torch.distributed.run on 127.0.0.1).  With fewer GPUs than N the ranks share them through
    the NCCL test shim and the line says so (functional check, not a timing)."""
    import torch
    env = dict(os.environ)
    ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if ndev < args.gpus and not env.get("TANQ_NCCL_LIB"):
        env["TANQ_NCCL_LIB"] = build_nccl_shim()
    # torch.distributed.run abbreviates its own options (--n would match --nnodes): pass the
    # script's options in unambiguous long form
    argv = ["--qubits" if a == "--n" else a for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd, env=env)


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and args.remap != "p2p":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # TANQ_NCCL_LIB = the NCCL test shim (tests/nccl_shim): ranks may share one GPU, the
    # torch-level plumbing runs on gloo; a functional check of the N > 1 path, not a timing
    shim = bool(os.environ.get("TANQ_NCCL_LIB"))
    dev = local % torch.cuda.device_count() if shim else local
    torch.cuda.set_device(dev)
    tdev = "cpu" if shim else "cuda"
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if shim:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from __graft_entry__ import build
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    import workloads as W
    from paper_2404_13184_b200 import Simulator, CReadout, nccl_unique_id
    from paper_2404_13184_b200.tanq import Plan

    c, nm = W.config_workload(args.config, n=args.n)
    n = c.n
    if world > 1:
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        sim = Simulator(n, world_size=world, rank=rank, device=dev, nccl_uid=uid[0])
    elif "WORLD_SIZE" in os.environ and args.shards == 1:  # torchrun N=1: the per-rank API
        sim = Simulator(n, world_size=1, rank=0, device=dev)
    else:  # one process: --shards virtual shards, or --remap p2p over --gpus devices
        sim = Simulator(n, args.shards)
    shards_total = world if world > 1 else args.shards
    stream = torch.cuda.Stream()          # a real stream: events on it bracket the kernels
    torch.cuda.set_stream(stream)
    sim.set_stream(stream.cuda_stream)
    ro = CReadout.of(nm)
    t_plan = time.perf_counter()
    # large states: the timed plan records per-launch CUDA events (the roofline's kernel times
    # come from the timed region itself; 2 events per ~10-20 ms launch cost nothing).  Small,
    # launch-bound states (< 1 GB, one shard): the timed plan replays as one CUDA graph and the
    # kernel times come from a separate profiled pass over the same steps.
    small = 16 * 4 ** n < (1 << 30) and shards_total == 1 and world == 1
    plan = Plan(sim, c, nm, fuse=args.fuse, k_max=args.kmax, profile=not small, graph=small)
    plan_wall_ms = (time.perf_counter() - t_plan) * 1e3
    pinfo = plan.info()
    try:
        counts = plan_counts(args.config, n, shards_total, args.fuse, args.kmax)
    except SystemExit:  # a size the committed table does not list: our arm counts live
        counts = {"gate_updates": pinfo["gate_updates"]}
    if pinfo["gate_updates"] != counts["gate_updates"]:
        raise SystemExit(f"workloads/plan_counts.json is stale ({counts['gate_updates']} vs "
                         f"{pinfo['gate_updates']} updates): run scripts/plan_counts.py")

    def step():
        sim.reset()
        st = plan.exec(sim)
        sim.probs(ro)
        return st

    for _ in range(args.warmup):
        st = step()
    sim.profile_reset()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(dev)
    clk.start()
    l0 = sim.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        st = step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    launches = sim.launch_count() - l0
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=tdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    ops = st["gate_updates"]          # fused-gate updates per step (a K3 group of m sub-ops = m)
    value = ops * args.steps / (ms / 1e3)
    prof_ms = ms
    if small:  # kernel times from a profiled pass of the same steps (not part of `value`)
        pplan = Plan(sim, c, nm, fuse=args.fuse, k_max=args.kmax, profile=True)
        sim.profile_reset()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(args.steps):
            sim.reset()
            pplan.exec(sim)
            sim.probs(ro)
        q1.record(stream)
        torch.cuda.synchronize()
        prof_ms = q0.elapsed_time(q1)
    prof = {p["name"]: p for p in sim.profile()}
    info = sim.info()

    # dominant kernel: the gate class with the most device time
    gate = max((p for p in prof.values() if p["name"].startswith(("gate", "group"))),
               key=lambda p: p["total_ms"])
    avg_ms = gate["total_ms"] / gate["launches"]
    bytes_launch = gate["bytes"] / gate["launches"]
    flops_launch = gate["flops"] / gate["launches"]
    hw_flops_launch = gate["hw_flops"] / gate["launches"]
    peak_gbs, peak_kind = measured_peaks()
    gbs = bytes_launch / (avg_ms * 1e-3) / 1e9
    share = gate["total_ms"] / prof_ms if prof_ms > 0 else None
    hbm_total = sum(p["bytes"] for p in prof.values())
    traffic, traffic_src = ncu_traffic(gate["name"], bytes_launch)
    # bound of the dominant kernel: the larger of its HBM floor (algorithmic bytes / measured
    # copy peak) and its FP64 floor (algorithmic flops / measured DMMA peak)
    peak_tf, peak_tf_kind = fp64_tensor_peak()
    tf = flops_launch / (avg_ms * 1e-3) / 1e12
    hw_tf = hw_flops_launch / (avg_ms * 1e-3) / 1e12
    t_hbm = bytes_launch / (peak_gbs * 1e9)
    t_fp = flops_launch / (peak_tf * 1e12)
    # the same launch in SURVEY §8(d)'s full-state basis: 32 B and 8 * 4^k flops per amplitude
    # of all 4^n / G amplitudes (the packed layout touches 16 B and does half of those flops)
    packed = gate["bytes"] > 0 and abs(bytes_launch / (16.0 * 2 ** info["local_bits"]) - 1) < 1e-9
    full_f = 2.0 if packed else 1.0
    full_basis = {
        "basis": "SURVEY §8(d) full state: 32 B and 8*4^k flops per amplitude of all 4^n/G "
                 "amplitudes per pass" + (" (2x the packed launch's own counts)" if packed else ""),
        "bytes_per_launch": bytes_launch * full_f, "flops_per_launch": flops_launch * full_f,
        "hbm_gbs_equiv": gbs * full_f, "hbm_frac_equiv": gbs * full_f / peak_gbs,
        "fp64_tflops_equiv": tf * full_f, "fp64_frac_equiv": tf * full_f / peak_tf}
    common = {"kernel": gate["name"], "traffic": traffic, "traffic_source": traffic_src,
              "algorithmic_bytes_per_launch": bytes_launch, "flops_per_launch": flops_launch,
              "avg_launch_ms": avg_ms, "launches": gate["launches"], "share_of_step": share,
              "hbm_gbs": gbs, "hbm_frac": gbs / peak_gbs, "hbm_peak": peak_gbs,
              "fp64_alg_tflops": tf, "fp64_frac": tf / peak_tf, "fp64_hw_tflops": hw_tf,
              "fp64_hw_frac": hw_tf / peak_tf, "fp64_peak": peak_tf,
              "fp64_peak_kind": peak_tf_kind,
              "floors_ms": {"hbm": t_hbm * 1e3, "fp64": t_fp * 1e3},
              "basis": ("packed Hermitian layout: 16 B per amplitude per pass and half the "
                        "flops (only the canonical element of each transpose pair is "
                        "processed)" if packed else "full layout: 32 B per amplitude per pass"),
              "full_state_basis": full_basis,
              "flops_note": "algorithmic flops = 8 per complex multiply-add; the DMMA kernels "
                            "execute 6 (3-multiply complex product)"}
    if t_fp > t_hbm:
        roofline = {"bound": "tensor", "achieved": tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": tf / peak_tf, "peak_kind": peak_tf_kind, **common}
    else:
        roofline = {"bound": "hbm", "achieved": gbs, "peak": peak_gbs, "unit": "GB/s",
                    "frac": gbs / peak_gbs,
                    "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)", **common}

    # ---- e2e: the public API from host objects, H2D of the inputs, D2H of the result ----
    # warm-up of the public path too: the first call plans (cache miss), the second captures
    # the plan's CUDA graph; only then is a call representative of a repeated run
    for _ in range(args.warmup):
        sim.reset()
        sim.run_circuit(c, nm, fuse=args.fuse, k_max=args.kmax)
        sim.probs(CReadout.of(nm))
    t_e2e, plan_ms_e2e = [], []
    for _ in range(max(1, args.steps)):
        torch.cuda.synchronize()
        a0 = time.perf_counter()
        sim.reset()
        st2 = sim.run_circuit(c, nm, fuse=args.fuse, k_max=args.kmax)
        p = sim.probs(CReadout.of(nm))
        torch.cuda.synchronize()
        t_e2e.append(time.perf_counter() - a0)
        plan_ms_e2e.append(st2["plan_ms"])
    e2e_s = statistics.median(t_e2e)
    if world > 1:
        t = torch.tensor([e2e_s], device=tdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = plan.h2d_bytes + sum(16 * (16 ** k) * st2[f"n_k{k}"] for k in (1, 2, 3))
    d2h = 8 * 2 ** n

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_estimate(args.config, n, ops, budget_s=args.ref_budget)
        cpu.pop("seconds", None)
        if args.whole_n:
            # the whole circuit at a small n, oracle end to end beside the GPU on the same plan
            wt, wp, wc, wnm = oracle_whole_circuit(args.config, args.whole_n)
            with Simulator(args.whole_n) as ws:
                ws.set_stream(stream.cuda_stream)
                wplan = Plan(ws, wc, wnm, fuse=args.fuse, k_max=args.kmax)
                for _ in range(3):
                    ws.reset()
                    wplan.exec(ws)
                reps = 20
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record(stream)
                for _ in range(reps):
                    ws.reset()
                    wst = wplan.exec(ws)
                    gp = ws.probs(CReadout.of(wnm))
                f1.record(stream)
                torch.cuda.synchronize()
                g_s = f0.elapsed_time(f1) / 1e3 / reps
            cpu["whole_circuit"] = {
                "n_qubits": args.whole_n, "basis_gates": len(wc.ops),
                "gate_updates": wst["gate_updates"], "oracle_s": wt, "gpu_s": g_s,
                "oracle_updates_per_s": wst["gate_updates"] / wt,
                "gpu_updates_per_s": wst["gate_updates"] / g_s,
                "max_abs_probs_diff": float(np.abs(gp - wp).max()),
                "note": "whole circuit, no sampling or scaling: the oracle end to end on all "
                        "host cores vs the GPU plan on the same circuit (readout-noisy probs "
                        "compared); at this n the GPU is launch-bound, so the ratio is a floor"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": (world if world > 1 else
                       min(args.shards, torch.cuda.device_count()) if args.remap == "p2p" else 1),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, c, counts),
            "parallelism": (f"{world} ranks sharing GPU(s) through the NCCL test shim "
                            f"(functional check, not a timing)" if shim and world > 1 else
                            f"state partitioned over {world} GPU(s) by high bits, one process "
                            f"per GPU, NCCL remaps" if world > 1 else
                            "1 GPU" if args.shards == 1 else
                            f"{args.shards} shards in one process over "
                            f"{min(args.shards, torch.cuda.device_count())} device(s), in-place "
                            f"peer-to-peer remap swaps (--remap p2p)" if args.remap == "p2p" else
                            f"{args.shards} virtual shards on 1 GPU (remap test mode)"),
            "plan": {"kernel_ops": st["ops_fused"],
                     "kernels_by_k": [st["n_k1"], st["n_k2"], st["n_k3"], st["n_k4"], st["n_k5"]],
                     "remaps_per_step": st["n_remaps"], "shard_bytes": info["shard_bytes"],
                     "plan_ms": pinfo["plan_ms"], "plan_wall_ms": plan_wall_ms,
                     "e2e_plan_ms": statistics.median(plan_ms_e2e)},
            "hbm_gbs": hbm_total / (prof_ms / 1e3) / 1e9,
            "amplitude_updates_per_s": value * 4 ** n,
            "circuit_gates_per_s": len(c.ops) * args.steps / (ms / 1e3),
            "roofline": roofline,
            "kernels": {k: {"launches": v["launches"], "avg_ms": v["total_ms"] / v["launches"],
                            "gbs": v["bytes"] / (v["total_ms"] * 1e-3) / 1e9,
                            "alg_tflops": v["flops"] / (v["total_ms"] * 1e-3) / 1e12,
                            "hw_tflops": v["hw_flops"] / (v["total_ms"] * 1e-3) / 1e12,
                            "share_of_step": v["total_ms"] / prof_ms}
                        for k, v in prof.items()},
            "kernel_timing": ("per-launch CUDA events on the library stream inside the timed region"
                              if not small else
                              "timed region replays the plan as one CUDA graph; per-kernel times "
                              "from a separate profiled pass of the same steps"),
            "cpu_baseline": cpu,
            "e2e": {"value": ops / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--qubits", "--n", dest="n", type=int, default=None,
                    help="qubits of the workload (--qubits under torchrun: it claims --n)")
    ap.add_argument("--fuse", type=int, default=2)
    ap.add_argument("--kmax", type=int, default=3)
    ap.add_argument("--ref-budget", type=float, default=8.0,
                    help="seconds of oracle work per cpu_baseline / reference step")
    ap.add_argument("--whole-n", type=int, default=None,
                    help="N=1: also run the whole config circuit at this n on the oracle beside "
                         "the GPU (default: 12 for config 4, else skipped; 0 = skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--remap", default="nccl", choices=["nccl", "p2p"],
                    help="--gpus N > 1: one process per GPU with NCCL point-to-point remaps "
                         "(torchrun) or one process holding all N shards with in-place P2P swap "
                         "kernels over peer memory")
    ap.add_argument("--shards", type=int, default=1,
                    help="N=1 only: split the state into this many virtual shards on the one GPU "
                         "(exercises the global-qubit remap with the in-place swap kernel)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.whole_n is None:
        args.whole_n = 12 if args.config == 4 else 0
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and args.remap == "p2p":
        args.shards = args.gpus
        return run_ours(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
