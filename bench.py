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
def oracle_sample(config: int, n_full: int, ops_fused: int, budget_s: float = 15.0):
    import numpy as np
    import workloads as W
    from oracle import channels, dense

    n_s = min(n_full, 13 if n_full > 14 else n_full)
    c_full, _ = W.config_workload(config, n=n_full)
    c, nm = W.config_workload(config, n=n_s)
    rho = dense.ground(n_s)
    dense.lib()
    t0 = time.perf_counter()
    done = 0
    for op in c.ops:
        dense.apply_channel_seq(rho, n_s, channels.gate_channel_sequence(op, nm))
        done += 1
        if time.perf_counter() - t0 > budget_s and done >= 2:
            break
    dt = time.perf_counter() - t0
    per_gate = dt / done * 4 ** (n_full - n_s)          # O(4^n) per gate
    t_circuit = per_gate * len(c_full.ops)
    value = ops_fused / t_circuit
    del rho
    sample = (f"oracle (oracle/dense.c, OpenMP) applied the first {done} of {len(c.ops)} "
              f"basis gates (noise channels unfused) of the same {config=} workload at n={n_s} "
              f"in {dt:.2f} s; per-gate time scaled by 4^({n_full}-{n_s}) to n={n_full} and "
              f"multiplied by the {len(c_full.ops)} gates of the full circuit "
              f"({t_circuit:.1f} s); value = the GPU plan's fused-gate updates per circuit / that time")
    return {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "sample": sample, "seconds": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import workloads as W
    c, nm = W.config_workload(args.config, n=args.n)
    # the fused op count the GPU arm executes per circuit (host planner, no GPU needed)
    ops_fused = fused_count_host(c, nm, args)
    vals = []
    t0 = time.perf_counter()
    cb = None
    for _ in range(args.steps):
        cb = oracle_sample(args.config, c.n, ops_fused, budget_s=args.ref_budget)
        vals.append(cb["value"])
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES.get(args.config, str(args.config)),
                       "n_qubits": c.n, "gates": len(c.ops), "gate_updates": ops_fused},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb["cores"],
                             "kind": "oracle", "sample": cb["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def fused_count_host(c, nm, args) -> int:
    """Fused op count of the GPU arm's plan (host planner only, no device work)."""
    from paper_2404_13184_b200.tanq import Plan
    p = Plan(None, c, nm, fuse=args.fuse, k_max=args.kmax, world_size=args.gpus)
    return p.info()["gate_updates"]


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
    if world != args.gpus:
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
    else:
        sim = Simulator(n, args.shards)
    stream = torch.cuda.Stream()          # a real stream: events on it bracket the kernels
    torch.cuda.set_stream(stream)
    sim.set_stream(stream.cuda_stream)
    ro = CReadout.of(nm)
    plan = Plan(sim, c, nm, fuse=args.fuse, k_max=args.kmax, profile=True)

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
    share = gate["total_ms"] / ms if ms > 0 else None
    hbm_total = sum(p["bytes"] for p in prof.values())
    traffic, traffic_src = ncu_traffic(gate["name"], bytes_launch)
    # bound of the dominant kernel: the larger of its HBM floor (algorithmic bytes / measured
    # copy peak) and its FP64 floor (algorithmic flops / measured DMMA peak)
    peak_tf, peak_tf_kind = fp64_tensor_peak()
    tf = flops_launch / (avg_ms * 1e-3) / 1e12
    hw_tf = hw_flops_launch / (avg_ms * 1e-3) / 1e12
    t_hbm = bytes_launch / (peak_gbs * 1e9)
    t_fp = flops_launch / (peak_tf * 1e12)
    common = {"kernel": gate["name"], "traffic": traffic, "traffic_source": traffic_src,
              "algorithmic_bytes_per_launch": bytes_launch, "flops_per_launch": flops_launch,
              "avg_launch_ms": avg_ms, "launches": gate["launches"], "share_of_step": share,
              "hbm_gbs": gbs, "hbm_frac": gbs / peak_gbs, "hbm_peak": peak_gbs,
              "fp64_alg_tflops": tf, "fp64_frac": tf / peak_tf, "fp64_hw_tflops": hw_tf,
              "fp64_hw_frac": hw_tf / peak_tf, "fp64_peak": peak_tf,
              "fp64_peak_kind": peak_tf_kind,
              "floors_ms": {"hbm": t_hbm * 1e3, "fp64": t_fp * 1e3},
              "flops_note": "algorithmic flops = 8 per complex multiply-add; the DMMA kernels "
                            "execute 6 (3-multiply complex product); packed-layout launches "
                            "count 16 B and half the flops per amplitude"}
    if t_fp > t_hbm:
        roofline = {"bound": "tensor", "achieved": tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": tf / peak_tf, "peak_kind": peak_tf_kind, **common}
    else:
        roofline = {"bound": "hbm", "achieved": gbs, "peak": peak_gbs, "unit": "GB/s",
                    "frac": gbs / peak_gbs,
                    "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)", **common}

    # ---- e2e: the public API from host objects, H2D of the inputs, D2H of the result ----
    t_e2e = []
    for _ in range(max(1, args.steps)):
        torch.cuda.synchronize()
        a0 = time.perf_counter()
        sim.reset()
        st2 = sim.run_circuit(c, nm, fuse=args.fuse, k_max=args.kmax)
        p = sim.probs(CReadout.of(nm))
        torch.cuda.synchronize()
        t_e2e.append(time.perf_counter() - a0)
    e2e_s = statistics.median(t_e2e)
    if world > 1:
        t = torch.tensor([e2e_s], device=tdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = plan.h2d_bytes + sum(16 * (16 ** k) * st2[f"n_k{k}"] for k in (1, 2, 3))
    d2h = 8 * 2 ** n

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(args.config, n, ops, budget_s=args.ref_budget)
        cpu.pop("seconds", None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES.get(args.config, str(args.config)),
                       "n_qubits": n, "gates": len(c.ops), "gate_updates": ops,
                       "kernel_ops": st["ops_fused"],
                       "fusion": f"fuse={args.fuse} k_max={args.kmax}",
                       "kernels_by_k": [st["n_k1"], st["n_k2"], st["n_k3"], st["n_k4"]],
                       "remaps_per_step": st["n_remaps"],
                       "state_bytes": 16 * 4 ** n, "shard_bytes": info["shard_bytes"],
                       "parallelism": (f"{world} ranks sharing GPU(s) through the NCCL test shim "
                                       f"(functional check, not a timing)" if shim and world > 1 else
                                       f"state partitioned over {world} GPU(s) by high bits"
                                       if args.shards == 1 else
                                       f"{args.shards} virtual shards on 1 GPU (remap test mode)"),
                       "l2": "inputs larger than L2 (state >> 126 MB)" if 16 * 4 ** n > 5e8
                       else "state fits L2 (no flush)"},
            "hbm_gbs": hbm_total / (ms / 1e3) / 1e9,
            "amplitude_updates_per_s": value * 4 ** n,
            "circuit_gates_per_s": len(c.ops) * args.steps / (ms / 1e3),
            "roofline": roofline,
            "kernels": {k: {"launches": v["launches"], "avg_ms": v["total_ms"] / v["launches"],
                            "gbs": v["bytes"] / (v["total_ms"] * 1e-3) / 1e9,
                            "alg_tflops": v["flops"] / (v["total_ms"] * 1e-3) / 1e12,
                            "hw_tflops": v["hw_flops"] / (v["total_ms"] * 1e-3) / 1e12,
                            "share_of_step": v["total_ms"] / ms}
                        for k, v in prof.items()},
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
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shards", type=int, default=1,
                    help="N=1 only: split the state into this many virtual shards on the one GPU "
                         "(exercises the global-qubit remap with the in-place swap kernel)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
