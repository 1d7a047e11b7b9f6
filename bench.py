#!/usr/bin/env python
"""Benchmark of the local-smoothing GMG hot path on B200 (BASELINE.json metric:
V-cycle DoFs/s and level-vmult HBM GB/s as a fraction of peak).

A step is one V-cycle preconditioner application x = V(b) (P:318-327 with local
smoothing) on the config-3 forest (3D Poisson, Q2, sphere-refined,
49.8M leaf DoFs, 11 levels), b uniform[-1,1) by canonical index, resident in
HBM.  DoFs = all leaf nodes (reading R22).  Inputs are larger than L2 (every
multigrid-layout vector is 466 MB > 126 MB), so no flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3] [--profile]

N > 1 (torchrun, one rank per GPU): the same forest is sharded along the SFC
partition with the first-child rule; every level exchanges ghosts with grouped
ncclSend/ncclRecv and CG dots use ncclAllReduce (strong scaling: total work
fixed).  --impl reference times the CPU oracle (oracle/, numpy/scipy, as it
stands) on a bounded sample of the same workload family (c3 recipe truncated at
4 passes).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "V-cycle DoFs/s and level vmult HBM GB/s (fraction of peak) at 1/2/4/8 B200"
UNIT = "DoFs/s"
WORKLOADS = {
    "c3": "BASELINE configs[2]: 3D Poisson -Laplace u = f on [0,1]^3, Q2, fp64, Dirichlet; 3 global "
          "refinements + 7 sphere-surface passes (|x-(.5,.5,.5)| = 0.3), 2:1 vertex balanced",
    "c2": "BASELINE configs[1]: 2D L-shape Q2, corner-graded to ~1M DoFs",
    "c3p4": "c3 recipe truncated at 4 passes (774,181 DoFs)",
    "c4": "BASELINE configs[3]: 3D -div(a grad u) = 1 on [0,1]^3, Q2, fp64, a log-uniform in [1e-2,1e2] per "
          "level-2 cell; corner-graded toward (0,0,0), s = 6, lmax = 19 (107M DoFs, 20 levels)",
    "c5": "BASELINE configs[4]: the c3 sphere forest with a shell half-width w_n (2^-10 units) giving "
          ">= 125M DoFs per GPU (weak scaling)",
}
SAMPLE = "c3p4"


def load_traffic(config, precision):
    """DRAM bytes per launch of the dominant kernel from a committed ncu capture
    (tools/traffic_from_ncu.py -> profiles/*_traffic.json), else None."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")), reverse=True):
        with open(p) as fh:
            e = json.load(fh).get(f"{config}/{precision}")
        if e:
            return e["traffic_bytes"], os.path.relpath(p, ROOT)
    return None, None


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.12)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        time.sleep(0.06)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        import statistics
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- reference arm
def oracle_sample(steps: int, warmup: int):
    """The oracle V-cycle, as it stands, on the bounded sample (c3 recipe at 4 passes)."""
    from gmg_inputs import config, uniform_pm1
    from oracle import forest as F, mg
    cfg = config(SAMPLE)
    t0 = time.time()
    f = F.generate(cfg)
    h = mg.build(f, cfg["k"])
    setup = time.time() - t0
    b = uniform_pm1(h.leaf.n_free)
    n_dofs = int(h.leaf.X.shape[0])
    for _ in range(warmup):
        mg.vcycle(h, b)
    t0 = time.perf_counter()
    for _ in range(steps):
        mg.vcycle(h, b)
    dt = (time.perf_counter() - t0) / max(steps, 1)
    return dict(value=n_dofs / dt, sec_per_vcycle=dt, n_dofs=n_dofs, setup_s=setup)


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    r = oracle_sample(args.steps, args.warmup)
    cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"{SAMPLE}: c3 recipe at 4 passes, {r['n_dofs']} DoFs, one V-cycle per step "
                     f"(scipy CSR level matrices, single thread), setup {r['setup_s']:.1f}s excluded"}
    out = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * r["sec_per_vcycle"], "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": WORKLOADS[SAMPLE], "sample_of": args.config},
           "cpu_baseline": cpu,
           "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1904_03317_b200 as G
    from gmg_inputs import config, uniform_pm1

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.config == "c5":
        from gmg_inputs import config_c5
        cfg = config_c5(world)
    else:
        cfg = config(args.config)
    t0 = time.time()
    f = G.gmg_forest_generate(G.recipe_from_config(cfg))
    part = G.gmg_partition(f, world, mode=args.partition)
    comm = None
    if world > 1:
        uid = [G.gmg_nccl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = G.NcclComm(uid[0], world, rank)
    mixed = args.precision == "mixed"
    coef = None
    if cfg.get("coef") == "level2_log_uniform":        # config 4: a per level-2 cell (SFC order)
        from gmg_inputs import log_uniform_coef
        coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"]))
    h = G.gmg_setup(f, part, k=cfg["k"], rank=rank, comm=comm, mixed=mixed, coef_level2=coef)
    setup_s = time.time() - t0
    info = h.info()
    n_dofs = info["n_leaf_nodes"]
    fo, n_own = info["first_owned"], info["n_owned"]
    canon = h.leaf_dofs()[3]
    b_can = uniform_pm1(info["n_leaf_free"])
    b = torch.tensor(b_can[canon[fo:fo + n_own]], device=dev, dtype=torch.float64)
    x = torch.zeros_like(b)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world > 1:
            tt = torch.tensor([v], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            v = float(tt.item())
        return v

    for _ in range(max(args.warmup, 1)):
        h.vcycle(b, x)
    barrier()
    if args.profile:
        torch.cuda.profiler.start()
        h.vcycle(b, x)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    launches0 = h.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            h.vcycle(b, x)
        e1.record(stream)
        e1.synchronize()
        barrier()
    launches = h.launch_count() - launches0
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    value = n_dofs * args.steps / t_dev            # one sharded V-cycle of the whole forest per step

    # ---- roofline of the dominant kernel: level operator on the finest level (rank-local)
    L = info["n_levels"] - 1
    fo_l, no_l, gh_l = h.rank_level(L)
    n_loc = no_l + len(gh_l)
    nL = info["level_dofs"][L]
    ncell = info["level_cells"][L]
    nn = (cfg["k"] + 1) ** cfg["dim"]
    vdt = torch.float32 if mixed else torch.float64
    xa = torch.tensor(uniform_pm1(n_loc), device=dev, dtype=vdt)
    ya = torch.zeros_like(xa)
    for _ in range(3):
        h.level_apply_kernel(L, xa, ya)
    reps = 20
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a0.record(stream)
    for _ in range(reps):
        h.level_apply_kernel(L, xa, ya)           # the kernel alone (no memset, no exchange)
    a1.record(stream)
    a1.synchronize()
    t_apply = max_over_ranks(a0.elapsed_time(a1) / 1e3 / reps)
    # 16 B per level DoF (x read, y write) + 4 B x 27 index entries per cell
    # (fp32 vectors in the mixed-precision V-cycle: 8 B per level DoF)
    vb = 4 if mixed else 8
    alg_bytes = (2 * vb * nL + 4 * nn * ncell) / world
    peak, peak_src = load_peaks()
    achieved = alg_bytes / t_apply / 1e9
    applies_per_vc = 2 * args.cheb_degree         # (m-1) pre + 1 residual + m post on every level
    share = applies_per_vc * t_apply / (t_dev / args.steps)

    # ---- end to end through the C ABI with host buffers (pinned), copies timed.
    # Every step copies its right-hand side host -> device, runs gmg_vcycle and
    # copies the result device -> host.  The copies run on their own streams,
    # double-buffered, so step i+1's upload and step i-1's download overlap
    # V-cycle i (copy engines vs SMs); the timed region starts before the first
    # upload and ends after the last download.
    nbuf = 2
    bh = [torch.tensor(b_can[canon[fo:fo + n_own]], dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    xh = [torch.empty(n_own, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    bd = [torch.empty_like(b) for _ in range(nbuf)]
    xd = [torch.empty_like(b) for _ in range(nbuf)]
    up, down = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev = {k: [torch.cuda.Event() for _ in range(nbuf)] for k in ("up", "vc", "down")}

    def e2e_run(n_steps, start=None):
        for q in range(nbuf):             # buffers free at the start
            ev["vc"][q].record(stream)
            ev["down"][q].record(stream)
        if start is not None:
            start.record(stream)
        up.wait_stream(stream)
        down.wait_stream(stream)
        for i in range(n_steps):
            q = i % nbuf
            up.wait_event(ev["vc"][q])                    # V-cycle i-2 has read bd[q]
            with torch.cuda.stream(up):
                bd[q].copy_(bh[q], non_blocking=True)
            ev["up"][q].record(up)
            stream.wait_event(ev["up"][q])
            stream.wait_event(ev["down"][q])              # xd[q] downloaded (step i-2)
            h.vcycle(bd[q], xd[q], stream=stream.cuda_stream)
            ev["vc"][q].record(stream)
            down.wait_event(ev["vc"][q])
            with torch.cuda.stream(down):
                xh[q].copy_(xd[q], non_blocking=True)
            ev["down"][q].record(down)
        for q in range(nbuf):
            stream.wait_event(ev["down"][q])

    e2e_run(2)
    barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(2, min(args.steps, 20))
    e2e_run(e2e_steps, start=s0)
    s1.record(stream)
    s1.synchronize()
    t_e2e = max_over_ranks(s0.elapsed_time(s1) / 1e3)
    e2e_value = n_dofs * e2e_steps / t_e2e
    # the downloaded result equals the device-resident V-cycle's
    e2e_check = float((xh[(e2e_steps - 1) % nbuf].to(dev) - xd[(e2e_steps - 1) % nbuf]).abs().max())

    # ---- one GMG-CG solve (context, not the metric)
    bb = torch.zeros_like(b)
    h.rhs_constant(1.0, bb)
    xs = torch.zeros_like(b)
    barrier()
    c0 = time.perf_counter()
    its, relres, _ = h.solve_cg(bb, xs, rtol=1e-8)
    torch.cuda.synchronize()
    t_cg = max_over_ranks(time.perf_counter() - c0)

    per_vc, per_la = h.launch_profile()
    traffic, traffic_src = load_traffic(args.config, args.precision) if world == 1 else (None, None)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_sample(steps=3, warmup=1)
        cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{SAMPLE}: c3 recipe at 4 passes, {r['n_dofs']} DoFs, 3 oracle V-cycles "
                         f"(scipy CSR, single thread), setup excluded"}
    if rank == 0:
        model = part.model()
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
               "scaling": "weak" if args.config == "c5" else "strong", "vs_baseline": None,
               "dtype": "f32" if mixed else "f64", "data": "synthetic",
               "config": {"workload": WORKLOADS.get(args.config, args.config), "config": args.config,
                          "precision": "fp32 V-cycle in fp64 CG" if mixed else "fp64",
                          "n_leaf_dofs": n_dofs, "n_free_dofs": info["n_leaf_free"], "levels": info["n_levels"],
                          "level_dofs": info["level_dofs"], "k": cfg["k"], "dim": cfg["dim"],
                          "cheb_degree": args.cheb_degree, "global_batch": 1,
                          "l2": "inputs larger than L2 (MG-layout vectors %.0f MB each > 126 MB)"
                                % (info["mg_vector_len"] * 8 / 1e6),
                          "parallelism": "single GPU" if world == 1 else
                          f"{world} ranks, SFC partition + first-child rule, NCCL ghost exchange",
                          "partition": args.partition, "partition_eta": model["eta"],
                          "ghost_children_ratio": sum(model["ghost_children"]) / max(sum(model["children"]), 1),
                          "setup_s": round(setup_s, 2)},
               "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                            "frac": achieved / peak, "traffic": traffic,
                            "traffic_source": traffic_src if traffic is not None else None,
                            "kernel": ("fam_tensor_apply<3,%d,%s>" if cfg["dim"] == 3 else "fam_tensor_apply2d<%d,%s>")
                                      % (cfg["k"], "float" if mixed else "double") + " (level operator), finest level",
                            "algorithmic_bytes_per_launch": alg_bytes, "launch_s": t_apply,
                            "share_of_step": share,
                            "share_definition": "8 finest-level operator passes per V-cycle x this kernel's "
                                                "launch time / step time (the fused variants of those "
                                                "passes do more work: profiles/r01_launches_*.txt)",
                            "peak_source": peak_src},
               "cpu_baseline": cpu,
               "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * info["n_leaf_free"],
                       "d2h_bytes_per_step": 8 * info["n_leaf_free"], "steps": e2e_steps,
                       "copies": "pinned, own streams, double-buffered (overlap the V-cycle)",
                       "max_abs_diff_host_vs_device": e2e_check},
               "gpu_launches": launches,
               "launches_per_vcycle": per_vc,
               "clocks": clk.summary(),
               "cg": {"iters": its, "rel_res": relres, "seconds": t_cg, "rtol": 1e-8,
                      "dofs_per_s": n_dofs / t_cg}}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        if comm is not None:
            del h
            comm.destroy()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--cheb-degree", type=int, default=4)
    ap.add_argument("--partition", default="first_child", choices=["first_child", "per_level"],
                    help="level ownership: first-child rule (P:604, default) or per-level SFC balance (P:597)")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "mixed"],
                    help="fp64 V-cycle (default, BASELINE) or fp32 V-cycle inside the fp64 CG (P:897)")
    ap.add_argument("--profile", action="store_true", help="cudaProfilerStart/Stop around one V-cycle")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and not args.profile:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
