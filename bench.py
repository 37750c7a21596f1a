#!/usr/bin/env python
"""Benchmark: Trotter steps/s of the grouped hot path (BASELINE.json metric).

Workload (default): BASELINE config 4 -- 1D XXZ chain, n=30 complex128
(16 GiB state), Jxy=1, Jz=0.5, h_i ~ U[-1,1] seed 3, Neel initial state,
first-order Trotter dt=0.01; greedy grouping + reference Clifford synthesis.
A "step" is one Trotter step (every group: C_j, exp(-i dt Lambda_j), C_j^+).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank drives one GPU (see DESIGN.md §7 for the sharded
path); rank 0 prints one JSON line. `--impl reference` times the reference's
own CPU implementation (oracle/_ref, compiled from the reference sources)
on the host cores.
"""
from __future__ import annotations

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

CONFIG_DESC = {
    1: "XXX chain n=16 PBC, Neel, order 1, dt=0.01",
    2: "2D TFIM 5x5 open, |+>^25, Suzuki S2, dt=0.02",
    3: "random 4-local n=28 M=2000, random_state(28,2), order 1, dt=0.005",
    4: "XXZ chain n=30 PBC Jxy=1 Jz=0.5, Neel, order 1, dt=0.01",
    5: "JW-style n=33, |1^16 0^17>, order 1, dt=0.01",
}
METRIC = "Trotter steps/s at n=30 complex128; achieved HBM GB/s per GPU vs peak"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    """dram bytes per tile-pass launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_tile_pass_summary.json")
    try:
        with open(p) as f:
            return float(json.load(f)["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for nm, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ workload

def build_workload(cfg: int, n: int):
    import paper_2206_11664_b200 as S
    from paper_2206_11664_b200 import models as M

    text = M.config_text(cfg, None if n == M.CONFIGS[cfg]["n"] else n)
    H = S.Hamiltonian.load(text)
    groups = S.partition_and_diagonalize(H)
    return text, H, groups


def init_state(psi, cfg: int, n: int, rank: int):
    from paper_2206_11664_b200 import models as M
    import paper_2206_11664_b200._capi as A

    init = M.CONFIGS[cfg]["init"]
    if init[0] == "basis":
        psi.set_basis(M.initial_index(cfg, n))
    elif init[0] == "plus":
        A.check(A.sd_state_set_plus(psi._s))
    else:
        A.check(A.sd_state_set_random(psi._s, init[1]))


# ------------------------------------------------------- CPU reference

def ref_step_seconds(ref, text, n, cfg, steps=1):
    """Wall time of `steps` reference Trotter steps (oracle/_ref) at n."""
    import numpy as np
    from paper_2206_11664_b200 import models as M

    h, nn, _ = ref.partition_text(text, synthesize=True)
    try:
        psi = np.zeros(1 << n, np.complex128)
        init = M.CONFIGS[cfg]["init"]
        if init[0] == "basis":
            psi[M.initial_index(cfg, n)] = 1.0
        elif init[0] == "plus":
            psi[:] = 1.0 / math.sqrt(1 << n)
        else:
            psi = ref.random_state(n, init[1])
        t0 = time.perf_counter()
        out, stats = ref.evolve_grouped(h, psi, n, M.CONFIGS[cfg]["dt"], steps, M.CONFIGS[cfg]["order"])
        dt = time.perf_counter() - t0
        return dt / steps, stats
    finally:
        ref.free(h)


def cpu_reference(cfg: int, n_target: int, budget_s: float = 30.0):
    """Reference CPU steps/s at n_target, measured on the largest n whose
    single step fits ~budget_s, scaled to n_target by state size x sweeps
    (the reference's step cost is linear in both)."""
    from oracle import oracle as O
    from paper_2206_11664_b200 import models as M

    ref = O.ref()
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    n_probe = min(n_target, 20)
    t_probe, st_probe = ref_step_seconds(ref, M.config_text(cfg, n_probe if n_probe != M.CONFIGS[cfg]["n"] else None),
                                         n_probe, cfg)
    sweeps = lambda st, n: (st["amp_reads"] + st["amp_writes"]) / (2.0 * (1 << n))
    n_run = n_probe
    for cand in range(n_target, n_probe, -1):
        est = t_probe * (1 << (cand - n_probe)) * 1.15
        if est <= budget_s:
            n_run = cand
            break
    if n_run != n_probe:
        text = M.config_text(cfg, None if n_run == M.CONFIGS[cfg]["n"] else n_run)
        t_run, st_run = ref_step_seconds(ref, text, n_run, cfg)
    else:
        t_run, st_run = t_probe, st_probe
    p_run = sweeps(st_run, n_run)
    if n_run == n_target:
        t_target = t_run
        sample = f"1 full reference Trotter step of config {cfg} at n={n_run} ({p_run:.0f} sweeps)"
    else:
        # sweeps/step at the target n from the reference's own schedule
        _, _, g = ref.partition_text(M.config_text(cfg, None if n_target == M.CONFIGS[cfg]["n"] else n_target))
        per = 0.0
        for gr in g:
            runs = len({c for c, _ in gr.cnots}) if gr.cnots else 0
            per += 2 * (len(gr.h_pre) + len(gr.h_post) + 0.5 * runs + (1 if (gr.czs or gr.s_layer) else 0)) + 1
        p_target = per * (2 if M.CONFIGS[cfg]["order"] == 2 else 1)
        t_target = t_run * (1 << (n_target - n_run)) * (p_target / p_run)
        sample = (f"1 full reference Trotter step of config {cfg} at n={n_run} ({p_run:.0f} sweeps, {t_run:.2f} s),"
                  f" scaled x2^{n_target - n_run} state size x {p_target:.0f}/{p_run:.0f} sweeps to n={n_target}")
    return {"value": 1.0 / t_target, "unit": "Trotter steps/s", "cores": threads, "kind": "reference",
            "sample": sample, "s_per_step": t_target,
            "host": _host_desc(), "omp_threads": int(os.environ.get("OMP_NUM_THREADS", threads)),
            "n_sample": n_run, "scale_to_target": t_target / t_run}


def _host_desc():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        d = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                d[k.strip()] = v.strip()
        return f"{d.get('Model name', '?')}; sockets={d.get('Socket(s)', '?')} cores/socket={d.get('Core(s) per socket', '?')} threads={d.get('CPU(s)', '?')}"
    except Exception:
        return "unknown"


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    from paper_2206_11664_b200 import models as M

    from oracle import oracle as O

    cfg, n = args.config, args.n
    K, W = max(1, args.steps), max(0, args.warmup)
    # each step is one reference Trotter step at the largest n whose step fits
    # the per-step budget (the whole K + W run stays within a few minutes),
    # scaled to n by state size x sweeps; the sizing run counts as a warm-up
    per_step = max(2.0, min(args.ref_budget, 180.0 / (K + W)))
    cb = cpu_reference(cfg, n, budget_s=per_step)
    ref = O.ref()
    n_s = cb["n_sample"]
    text = M.config_text(cfg, None if n_s == M.CONFIGS[cfg]["n"] else n_s)
    for _ in range(W - 1):
        ref_step_seconds(ref, text, n_s, cfg)
    times = [ref_step_seconds(ref, text, n_s, cfg)[0] * cb["scale_to_target"] for _ in range(K)]
    v = K / sum(times)
    cb = dict(cb, value=v, s_per_step=sum(times) / K,
              sample=cb["sample"] + f"; {K} timed samples after {W} warm-up")
    line = {
        "metric": METRIC, "value": v, "unit": "Trotter steps/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": 1000.0 / v, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128 (f64 pairs)", "data": "synthetic (seeded generator, BASELINE config)",
        "config": {"workload": f"config{cfg}: {CONFIG_DESC[cfg]}", "n_qubits": n, "dt": M.CONFIGS[cfg]["dt"],
                   "order": M.CONFIGS[cfg]["order"]},
        "impl": "reference", "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "Trotter steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ our arm

def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2206_11664_b200 as S
    from paper_2206_11664_b200 import models as M

    cfg, n = args.config, args.n
    dev = local_rank
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    text, H, groups = build_workload(cfg, n)
    dt = M.CONFIGS[cfg]["dt"]
    order = M.CONFIGS[cfg]["order"]
    # N > 1: the state is sharded on the top log2(N) qubits (one shard per
    # rank); qubit remaps run over NCCL inside sd_evolve.
    psi = S.StateVector(n, device=dev, rank=rank, world=world)
    if world > 1:
        import torch.distributed as dist
        uid = [S.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        psi.attach_comm(uid[0])
        if not args.nccl_exchange:
            # fused exchange: the pass in front of each remap stores straight
            # into the peers' buffers over NVLink (CUDA IPC mappings)
            handles = [None] * world
            dist.all_gather_object(handles, psi.ipc_handles())
            psi.attach_peers(handles)
    plan = S.TrotterPlan(psi, groups, order=order, tile_qubits=args.tile)
    init_state(psi, cfg, n, rank)

    plan.evolve(dt, args.warmup)
    info = plan.info()  # steady-state layout's schedule
    stream = torch.cuda.ExternalStream(psi.stream(), device=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    barrier()
    clk = ClockSampler(dev)
    clk.start()
    # Per-launch CUDA events inside the timed region give the roofline's kernel
    # times. Small unsharded states run each step as a CUDA graph (launch-bound
    # regime); events would disable that, so there the kernel split comes from
    # a short profiled run after the timed region.
    graph_steps = world == 1 and psi.n_local <= 20
    plan.set_profiling(not graph_steps)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    plan.evolve(dt, args.steps, wait=False)
    e1.record(stream)
    e1.synchronize()
    barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    if graph_steps:
        plan.set_profiling(True)
        plan.evolve(dt, min(args.steps, 10))
    kt = plan.kernel_times()
    plan.set_profiling(False)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    steps_per_s = 1000.0 / ms_per_step
    value = steps_per_s  # one state, sharded over all ranks: whole-job steps/s

    # norm check after warmup+timed steps (exact power-of-two normalisation)
    nsq = psi.norm_sq_local()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([nsq], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t)
        nsq = float(t.item())
    norm_err = abs(math.sqrt(nsq) - 1.0)

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        host = torch.empty(2 << psi.n_local, dtype=torch.float64, pin_memory=True)
        psi.download_ptr(host.data_ptr(), 1 << psi.n_local)
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        fu = torch.cuda.Event(enable_timing=True)
        fe = torch.cuda.Event(enable_timing=True)
        psi.upload_ptr(host.data_ptr(), 1 << psi.n_local)       # H2D of the step inputs
        fu.record(stream)
        plan.evolve(dt, args.steps, wait=False)
        fe.record(stream)
        psi.download_ptr(host.data_ptr(), 1 << psi.n_local)     # D2H of the result
        f1.record(stream)
        f1.synchronize()
        e2e_ms = f0.elapsed_time(f1)
        split_ms = {"h2d_ms": f0.elapsed_time(fu), "steps_ms": fu.elapsed_time(fe), "d2h_ms": fe.elapsed_time(f1)}
        bytes_state = 16 * (1 << psi.n_local)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e2e_ms], device=f"cuda:{dev}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": args.steps * 1000.0 / e2e_ms, "unit": "Trotter steps/s",
               "h2d_bytes_per_step": bytes_state / args.steps, "d2h_bytes_per_step": bytes_state / args.steps,
               "api": "StateVector.upload -> TrotterPlan.evolve(K steps) -> download (sd_state_upload/sd_evolve/sd_state_download)",
               "trotter_steps_per_call": args.steps, "rank0_split": split_ms}
        del host

    peak, peak_src = load_peaks()
    tp = kt["tile_pass"]
    dp = kt["diag_pass"]
    xp = kt["exchange"]
    launches = tp["launches"] + dp["launches"]
    tot_ms = tp["ms"] + dp["ms"]
    if graph_steps:  # kernel split from the short profiled run, scaled to the timed steps
        prof_steps = min(args.steps, 10)
        tot_ms *= args.steps / prof_steps
        launches = info["n_kernels_per_step"] * args.steps
    bytes_per_launch = 2.0 * 16.0 * (1 << psi.n_local)
    dom = tp if tp["ms"] >= dp["ms"] else dp
    achieved = (bytes_per_launch / ((dom["ms"] / max(1, dom["launches"])) / 1e3)) / 1e9 if dom["launches"] else 0.0
    step_gbs = info["bytes_per_step"] / (ms_per_step / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "Trotter steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "c128 (f64 pairs)", "data": "synthetic (seeded generator, BASELINE config)",
        "config": {"workload": f"config{cfg}: {CONFIG_DESC[cfg]}", "n_qubits": n, "dt": dt, "order": order,
                   "parallelism": (f"state sharded on the top {int(math.log2(world))} qubits; qubit remaps "
                                   + ("as NCCL send/recv" if args.nccl_exchange else
                                      "fused into the preceding pass (peer-memory stores over NVLink)"))
                   if world > 1 else "single GPU",
                   "exchanges_per_step": info["n_exchanges_per_step"],
                   "l2": "state (16 GiB at n=30) >> 126 MB L2; no flush needed",
                   "tile_qubits": info["tile_qubits"], "passes_per_step": info["n_passes_per_step"],
                   "ref_sweeps_per_step": info["n_ref_sweeps_per_step"],
                   "floor_group_applications": info["n_group_applications"]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": load_traffic(), "peak_source": peak_src,
                     "kernel": "fused Clifford/diagonal tile pass (sdb_pass: NVRTC-specialised per program for n_local >= 22; k_tile_pass interpreter otherwise)",
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "avg_launch_ms": dom["ms"] / max(1, dom["launches"]),
                     "step_hbm_gbs": step_gbs, "step_frac": step_gbs / peak,
                     "share_of_step": tot_ms / max(1e-9, ms),
                     "timing": ("timed region replays CUDA graphs; kernel split from a separate profiled run"
                                if graph_steps else "per-launch CUDA events inside the timed region")},
        "gpu_launches": int(launches),
        "nvlink": ({"exchanges": int(xp["launches"]), "ms": xp["ms"],
                    "achieved_gbs_per_direction": (xp["bytes"] / 2.0 / (xp["ms"] / 1e3) / 1e9) if xp["ms"] else None,
                    "peak_gbs_per_direction": 900.0} if world > 1 else None),
        "clocks": clocks,
        "norm_error": norm_err,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_reference(cfg, n, budget_s=args.ref_budget)
        except Exception as ex:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def run_baseline_method(args, rank, world, local_rank):
    """The paper's comparison method on the same GPU (evolve_baseline,
    evolve.cpp:21-32: one rotation sweep per term, Hamiltonian order), so the
    grouped-vs-per-term speedup of the paper can be
    reported on B200. Single GPU, unsharded."""
    import torch

    import paper_2206_11664_b200 as S
    from paper_2206_11664_b200 import models as M

    if rank != 0:
        return 0
    cfg, n = args.config, args.n
    torch.cuda.set_device(local_rank)
    text, H, groups = build_workload(cfg, n)
    dt = M.CONFIGS[cfg]["dt"]
    psi = S.StateVector(n, device=local_rank)
    init_state(psi, cfg, n, 0)
    plan = S.EvolutionPlan(total_time=dt * args.warmup, n_steps=args.warmup)
    S.evolve_baseline(H, psi, plan)
    stream = torch.cuda.ExternalStream(psi.stream(), device=local_rank)
    torch.cuda.synchronize(local_rank)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    S.evolve_baseline(H, psi, S.EvolutionPlan(total_time=dt * args.steps, n_steps=args.steps))
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    m = H.term_count()
    line = {"metric": METRIC, "value": 1000.0 / ms, "unit": "Trotter steps/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128 (f64 pairs)", "data": "synthetic (seeded generator, BASELINE config)",
            "config": {"workload": f"config{cfg}: {CONFIG_DESC[cfg]}", "n_qubits": n, "dt": dt,
                       "method": "evolve_baseline (per-term rotation sweeps, the paper's comparison method)",
                       "sweeps_per_step": m},
            "roofline": {"bound": "hbm", "step_hbm_gbs": 32.0 * (1 << n) * m / (ms / 1e3) / 1e9}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=30.0)
    ap.add_argument("--nccl-exchange", action="store_true",
                    help="N>1: qubit remaps as grouped ncclSend/ncclRecv instead of the fused peer-memory store")
    ap.add_argument("--method", choices=["grouped", "baseline"], default="grouped",
                    help="grouped (the hot path) or the paper's per-term baseline on the GPU")
    args = ap.parse_args()
    from paper_2206_11664_b200 import models as M
    if args.n is None:
        args.n = M.CONFIGS[args.config]["n"]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    if args.method == "baseline":
        return run_baseline_method(args, rank, world, local_rank)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
