#!/usr/bin/env python
"""Benchmark of the local-smoothing GMG hot path on B200 (BASELINE.json metric:
V-cycle DoFs/s and level-vmult HBM GB/s as a fraction of peak, 1/2/4/8 B200).

A step is one V-cycle preconditioner application x = V(b) (P:318-327 with local
smoothing) -- all SURVEY §8(a) rows of the cycle: Chebyshev-Jacobi
pre/post smoothing with the matrix-free level operator, residual with the edge
rows, restriction, coarse solve, prolongation, copy to/from the level vectors.
b is uniform[-1,1) by canonical index, resident in HBM.  DoFs = all leaf nodes
(reading R22).

Headline workload (N = 1): BASELINE configs[4], config 5, the largest
configuration that fits one GPU: the config-3 sphere forest widened to >= 125M
DoFs per GPU (weak scaling: N GPUs run the N-sized forest, >= 125M N DoFs,
sharded along the SFC with the first-child rule).  The same run also measures
config 3 (49.8M DoFs, the strong-scaling config) as "secondary".  Inputs are
larger than L2 (every multigrid-layout vector is >= 466 MB > 126 MB), so no L2
flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c5] [--secondary c3|none] [--transport nccl|host]

N > 1: launched by the driver under torchrun (one rank per GPU, NCCL); run
directly with --gpus N it re-launches itself under torchrun.  --transport host
joins the ranks through host shared memory instead of NCCL (gmg_host_world:
the multi-process flow on fewer GPUs than ranks, for correctness, never a
performance number).  --impl reference times the CPU oracle (oracle/, as it
stands) on a bounded sample of the same workload family.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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
          "refinements + 7 sphere-surface passes (|x-(.5,.5,.5)| = 0.3), 2:1 vertex balanced (49.8M DoFs)",
    "c2": "BASELINE configs[1]: 2D L-shape Q2, corner-graded to ~1M DoFs",
    "c3p4": "c3 recipe truncated at 4 passes (774,181 DoFs)",
    "c4": "BASELINE configs[3]: 3D -div(a grad u) = 1 on [0,1]^3, Q2, fp64, a log-uniform in [1e-2,1e2] per "
          "level-2 cell; corner-graded toward (0,0,0), s = 6, lmax = 19 (107M DoFs, 20 levels)",
    "c5": "BASELINE configs[4]: 3D Poisson weak scaling, Q2, fp64: the config-3 sphere forest refined on the "
          "shell |x-(.5,.5,.5)| in [0.3-w_n, 0.3+w_n], w_n the smallest multiple of 2^-10 giving >= 125M DoFs "
          "per GPU (reading R21)",
}
SAMPLE = "c3p4"
KIND_ORDER = ["res_restrict", "apply", "cheb_x1", "cheb_11", "cheb_10", "cheb_01", "cheb_00", "cheb_p01", "cheb_stream",
              "cheb_stream_full", "restrict", "prolongate", "coarse"]


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


def load_traffic(config, precision, kind, level):
    """DRAM bytes per launch of a kernel from a committed ncu --set full capture
    (tools/traffic_from_ncu.py -> profiles/*_traffic.json), else None."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")), reverse=True):
        with open(p) as fh:
            d = json.load(fh)
        for key in (f"{config}/{precision}/{kind}/{level}", f"{config}/{precision}/{kind}"):
            e = d.get(key)
            if e:
                return e["traffic_bytes"], os.path.relpath(p, ROOT)
    return None, None


def host_info():
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as fh:
            for ln in fh:
                if ln.startswith("MemTotal"):
                    ram = round(int(ln.split()[1]) / 1e6, 1)
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gb": ram}


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


# ---------------------------------------------------------------- the oracle (CPU baseline / reference arm)
def oracle_sample(steps: int, warmup: int, threads: int):
    """The oracle V-cycle, as it stands, on the bounded sample (c3 recipe at 4
    passes, 774,181 DoFs).  threads > 1: the row-parallel CSR matvec
    (oracle/spmv.py, bit-identical results)."""
    from gmg_inputs import config, uniform_pm1
    from oracle import forest as F, mg, spmv
    if threads > 1:
        try:
            spmv.build()
        except Exception:
            pass
    used = spmv.set_threads(threads)
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
    spmv.set_threads(1)
    return dict(value=n_dofs / dt, sec_per_vcycle=dt, n_dofs=n_dofs, setup_s=setup, threads=used, hier=h)


def oracle_timings(steps=3, warmup=1):
    """1 thread and all host cores on the same sample (the hierarchy is built once)."""
    from oracle import mg, spmv
    from gmg_inputs import uniform_pm1
    r1 = oracle_sample(steps, warmup, 1)
    h = r1.pop("hier")
    ncores = os.cpu_count() or 1
    try:
        spmv.build()
    except Exception:
        pass
    used = spmv.set_threads(ncores)
    b = uniform_pm1(h.leaf.n_free)
    mg.vcycle(h, b)
    t0 = time.perf_counter()
    for _ in range(steps):
        mg.vcycle(h, b)
    dt = (time.perf_counter() - t0) / steps
    spmv.set_threads(1)
    return r1, {"value": r1["n_dofs"] / dt, "sec_per_vcycle": dt, "threads": used}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    ncores = os.cpu_count() or 1
    r = oracle_sample(args.steps, args.warmup, ncores)
    r.pop("hier", None)
    hi = host_info()
    cpu = {"value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "oracle",
           "sample": f"{SAMPLE}: c3 recipe at 4 passes, {r['n_dofs']} DoFs, one oracle V-cycle per step "
                     f"(scipy CSR level matrices, row-parallel matvec on {r['threads']} threads, "
                     f"bit-identical to 1 thread), setup {r['setup_s']:.1f}s excluded", **hi}
    out = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * r["sec_per_vcycle"], "higher_is_better": True,
           "scaling": "weak" if args.config == "c5" else "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": WORKLOADS[SAMPLE], "sample_of": args.config, "n_leaf_dofs": r["n_dofs"]},
           "cpu_baseline": cpu,
           "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- our arm
class Ctx:
    """Per-process state shared by the measurements (ranks, device, comm)."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        import paper_1904_03317_b200 as G
        self.G, self.torch, self.dist = G, torch, dist
        self.rank, self.world, self.local = env_rank()
        if self.world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={self.world}")
        ndev = torch.cuda.device_count()
        if args.transport == "nccl" and self.world > ndev:
            raise SystemExit(f"{self.world} ranks need {self.world} GPUs for NCCL (found {ndev}); "
                             "use --transport host to run the multi-process flow on fewer GPUs")
        self.gpu = self.local % ndev
        torch.cuda.set_device(self.gpu)
        self.dev = torch.device("cuda", self.gpu)
        self.transport = args.transport
        self.comm = None
        if self.world > 1:
            if args.transport == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
                uid = [G.gmg_nccl_get_unique_id() if self.rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                self.comm = G.NcclComm(uid[0], self.world, self.rank)
            else:
                dist.init_process_group("gloo")
                name = [f"/gmg_bench_{os.getpid()}_{int(time.time())}" if self.rank == 0 else None]
                dist.broadcast_object_list(name, src=0)
                self.comm = G.HostWorld(name[0], self.world, self.rank)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, v):
        if self.world > 1:
            t = self.torch.tensor([v], dtype=self.torch.float64,
                                  device=self.dev if self.transport == "nccl" else "cpu")
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
            v = float(t.item())
        return v

    def close(self):
        if self.world > 1:
            self.dist.barrier()
            if self.comm is not None:
                self.comm.destroy()
            self.dist.destroy_process_group()


def kernel_table(recs, n_rep, step_s, peak, config, precision):
    """Per (kind, level): launch time (CUDA events on the launching stream), its
    algorithmic GB/s and fraction of the HBM peak, and its share of the step."""
    rows = []
    for r in recs:
        if r["kind"] in ("exchange", "copy_mg", "other", "leaf_apply") or r["launches"] == 0:
            continue
        t = r["seconds"] / r["launches"]
        if t <= 0:
            continue
        ach = r["bytes"] / t / 1e9
        rows.append({"kind": r["kind"], "level": r["level"], "launches_per_step": r["launches"] / n_rep,
                     "launch_us": 1e6 * t, "algorithmic_bytes": r["bytes"], "achieved_gbs": ach,
                     "frac": ach / peak, "layout_bytes": r["bytes_layout"],
                     "frac_layout": r["bytes_layout"] / t / 1e9 / peak,
                     "share_of_step": r["seconds"] / n_rep / step_s})
    rows.sort(key=lambda e: -e["share_of_step"])
    return rows


def time_level_vmult(ctx, h, info, L, mixed, peak, reps=10):
    """The plain level operator y = K_L x on the finest level (the paper's "level
    vmult") timed on its own through gmg_level_apply_kernel: the V-cycle
    has none since its residual runs fused with the restriction (TA_RES).  CUDA
    events around each launch on the launching stream; y is zeroed between
    launches outside the events.  Bytes as DESIGN.md section 6 (kind apply)."""
    torch = ctx.torch
    dt = torch.float32 if mixed else torch.float64
    vb = 4 if mixed else 8
    n = info["level_dofs"][L]
    k, dim = info["k"], info["dim"]
    nn, npch = (k + 1) ** dim, (2 * k + 1) ** dim
    g = torch.Generator(device=ctx.dev).manual_seed(190403317)
    xl = (2 * torch.rand(n, device=ctx.dev, dtype=torch.float64, generator=g) - 1).to(dt)
    yl = torch.zeros_like(xl)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        yl.zero_()
        h.level_apply_kernel(L, xl, yl)
    ts = []
    for _ in range(reps):
        yl.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h.level_apply_kernel(L, xl, yl)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = sum(ts) / len(ts)
    survey = 2.0 * vb * n + 4.0 * nn * info["level_cells"][L]
    layout = 2.0 * vb * n + 4.0 * npch * info["level_families"][L]
    return {"level": L, "launch_us": 1e6 * t, "achieved_gbs": survey / t / 1e9,
            "frac_survey_bytes": survey / t / 1e9 / peak, "frac_layout_bytes": layout / t / 1e9 / peak,
            "survey_bytes": survey, "layout_bytes": layout,
            "source": "gmg_level_apply_kernel on the finest level, %d launches (not in the V-cycle: "
                      "its residual is fused with the restriction)" % reps}


def measure(ctx, args, name, main=True):
    import numpy as np
    torch, G = ctx.torch, ctx.G
    from gmg_inputs import config, config_c5, uniform_pm1, log_uniform_coef
    cfg = config_c5(ctx.world) if name == "c5" else config(name)
    t0 = time.time()
    f = G.gmg_forest_generate(G.recipe_from_config(cfg))
    # N > 1: the smallest levels are gathered on rank 0
    part = G.gmg_partition(f, ctx.world, mode=args.partition, coarse_cells=args.coarse_cells if ctx.world > 1 else 0)
    mixed = args.precision == "mixed"
    coef = None
    if cfg.get("coef") == "level2_log_uniform":        # config 4: a per level-2 cell (SFC order)
        coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"]))
    # N > 1: rank-local setup (only this rank's part of the level topology,
    # P:529-539); inputs drawn by node key (independent of N)
    rank_local = ctx.world > 1
    h = G.gmg_setup(f, part, k=cfg["k"], rank=ctx.rank, comm=ctx.comm, mixed=mixed, coef_level2=coef,
                    cheb_degree=args.cheb_degree, device=ctx.gpu, rank_local=rank_local)
    setup_s = time.time() - t0
    info = h.info()
    n_dofs = info["n_leaf_nodes"]
    n_own = info["n_owned"]
    if rank_local:
        from gmg_inputs import uniform_pm1_keys
        b_host = np.ascontiguousarray(uniform_pm1_keys(h.owned_leaf_keys()[0]))
    else:
        fo = info["first_owned"]
        canon = h.leaf_dofs()[3]
        b_can = uniform_pm1(info["n_leaf_free"])
        b_host = np.ascontiguousarray(b_can[canon[fo:fo + n_own]])
        del canon, b_can
    b = torch.tensor(b_host, device=ctx.dev, dtype=torch.float64)
    x = torch.zeros_like(b)
    stream = torch.cuda.current_stream()

    for _ in range(max(args.warmup, 1)):
        h.vcycle(b, x)
    ctx.barrier()
    if args.profile and main:      # one V-cycle inside cudaProfilerStart/Stop (ncu --profile-from-start off)
        torch.cuda.profiler.start()
        h.vcycle(b, x)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    launches0 = h.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(ctx.gpu) as clk:
        ctx.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            h.vcycle(b, x)
        e1.record(stream)
        e1.synchronize()
        ctx.barrier()
    launches = h.launch_count() - launches0
    t_dev = ctx.max_over_ranks(e0.elapsed_time(e1) / 1e3)
    step_s = t_dev / args.steps
    value = n_dofs * args.steps / t_dev            # the whole forest, all ranks, per second

    # ---- per-kernel launch times (CUDA events around every launch of eager V-cycles)
    n_rep = 2
    recs = h.profile_vcycle(b, x, n_rep=n_rep)
    peak, peak_src = load_peaks()
    rows = kernel_table(recs, n_rep, step_s, peak, name, args.precision)
    L = info["n_levels"] - 1
    dom = rows[0]
    traffic, traffic_src = load_traffic(name, args.precision, dom["kind"], dom["level"]) \
        if ctx.world == 1 else (None, None)
    roofline = {"bound": "hbm", "achieved": dom["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "frac": dom["frac"], "traffic": traffic, "traffic_source": traffic_src,
                "kernel": f"{dom['kind']} (level {dom['level']})", "launch_s": dom["launch_us"] * 1e-6,
                "algorithmic_bytes_per_launch": dom["algorithmic_bytes"],
                "frac_layout_bytes": dom["frac_layout"], "share_of_step": dom["share_of_step"],
                "peak_source": peak_src,
                "definition": "dominant kernel = largest share of the step (gmg_profile_vcycle: CUDA events "
                              "around each launch of eager V-cycles on the launching stream); algorithmic "
                              "bytes per DESIGN.md §6 (operator: 2 vectors per level DoF + (k+1)^d int32 per "
                              "cell, SURVEY 8(d); fused Chebyshev: + the R1 rows' vectors); frac_layout_bytes "
                              "counts the (2k+1)^d patch rows the kernel reads instead"}
    plain = [r for r in rows if r["kind"] == "apply" and r["level"] == L]
    apply_plain = None
    if plain:
        a = plain[0]
        apply_plain = {"level": L, "launch_us": a["launch_us"], "achieved_gbs": a["achieved_gbs"],
                       "frac_survey_bytes": a["frac"], "frac_layout_bytes": a["frac_layout"],
                       "survey_bytes": a["algorithmic_bytes"], "layout_bytes": a["layout_bytes"],
                       "source": "V-cycle profile"}
    elif ctx.world == 1:
        apply_plain = time_level_vmult(ctx, h, info, L, mixed, peak)
    kernels = [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()} for r in rows[:10]]
    res = {"config": name, "n_leaf_dofs": n_dofs, "n_free_dofs": info["n_leaf_free"], "levels": info["n_levels"],
           "setup_s": round(setup_s, 2), "value": value, "ms_per_step": 1e3 * step_s, "gpu_launches": launches,
           "launches_per_vcycle": h.launch_profile()[0], "clocks": clk.summary(), "roofline": roofline,
           "apply_plain": apply_plain, "kernels": kernels, "info": info, "cfg": cfg}

    if main:
        # ---- end to end through the C ABI with host buffers (pinned), copies timed:
        # every step uploads its right-hand side, runs gmg_vcycle and downloads the
        # result; copies on their own streams, double-buffered (step i+1's upload and
        # step i-1's download overlap V-cycle i); the timed region starts before the
        # first upload and ends after the last download.
        nbuf = 2
        bh = [torch.from_numpy(b_host).pin_memory() for _ in range(nbuf)]
        xh = [torch.empty(n_own, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
        bd = [torch.empty_like(b) for _ in range(nbuf)]
        xd = [torch.empty_like(b) for _ in range(nbuf)]
        up, down = torch.cuda.Stream(device=ctx.dev), torch.cuda.Stream(device=ctx.dev)
        ev = {k: [torch.cuda.Event() for _ in range(nbuf)] for k in ("up", "vc", "down")}

        def e2e_run(n_steps, start=None):
            for q in range(nbuf):
                ev["vc"][q].record(stream)
                ev["down"][q].record(stream)
            if start is not None:
                start.record(stream)
            up.wait_stream(stream)
            down.wait_stream(stream)
            for i in range(n_steps):
                q = i % nbuf
                up.wait_event(ev["vc"][q])
                with torch.cuda.stream(up):
                    bd[q].copy_(bh[q], non_blocking=True)
                ev["up"][q].record(up)
                stream.wait_event(ev["up"][q])
                stream.wait_event(ev["down"][q])
                h.vcycle(bd[q], xd[q], stream=stream.cuda_stream)
                ev["vc"][q].record(stream)
                down.wait_event(ev["vc"][q])
                with torch.cuda.stream(down):
                    xh[q].copy_(xd[q], non_blocking=True)
                ev["down"][q].record(down)
            for q in range(nbuf):
                stream.wait_event(ev["down"][q])

        e2e_run(2)
        ctx.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_steps = max(2, min(args.steps, 20))
        e2e_run(e2e_steps, start=s0)
        s1.record(stream)
        s1.synchronize()
        t_e2e = ctx.max_over_ranks(s0.elapsed_time(s1) / 1e3)
        qlast = (e2e_steps - 1) % nbuf
        res["e2e"] = {"value": n_dofs * e2e_steps / t_e2e, "unit": UNIT,
                      "h2d_bytes_per_step": 8 * info["n_leaf_free"], "d2h_bytes_per_step": 8 * info["n_leaf_free"],
                      "steps": e2e_steps, "copies": "pinned, own streams, double-buffered (overlap the V-cycle)",
                      "max_abs_diff_host_vs_device": float((xh[qlast].to(ctx.dev) - xd[qlast]).abs().max())}
        del bh, xh, bd, xd

    # ---- one GMG-CG solve to 1e-8 (context, not the metric)
    bb = torch.zeros_like(b)
    h.rhs_constant(1.0, bb)
    xs = torch.zeros_like(b)
    ctx.barrier()
    c0 = time.perf_counter()
    its, relres, _ = h.solve_cg(bb, xs, rtol=1e-8)
    torch.cuda.synchronize()
    t_cg = ctx.max_over_ranks(time.perf_counter() - c0)
    res["cg"] = {"iters": its, "rel_res": relres, "seconds": t_cg, "rtol": 1e-8, "dofs_per_s": n_dofs / t_cg}
    model = part.model()
    res["partition_eta"] = model["eta"]
    res["setup"] = "rank-local (GMG_RANK_LOCAL)" if rank_local else "global numbering"
    res["ghost_children_ratio"] = sum(model["ghost_children"]) / max(sum(model["children"]), 1)
    res["mg_vector_mb"] = info["mg_vector_len"] * (4 if mixed else 8) / 1e6
    h.close()
    del b, x, bb, xs
    torch.cuda.empty_cache()
    return res


def run_ours(args):
    ctx = Ctx(args)
    main = measure(ctx, args, args.config, main=True)
    sec = None
    if args.secondary not in ("none", args.config):
        sec = measure(ctx, args, args.secondary, main=False)
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        r1, rall = oracle_timings(steps=3, warmup=1)
        cpu = {"value": rall["value"], "unit": UNIT, "cores": rall["threads"], "kind": "oracle",
               "value_1_thread": r1["value"],
               "sample": f"{SAMPLE}: c3 recipe at 4 passes, {r1['n_dofs']} DoFs, 3 oracle V-cycles (scipy CSR "
                         f"level matrices; row-parallel matvec on {rall['threads']} threads, bit-identical to "
                         f"the 1-thread run also given), setup excluded", **host_info()}
    if ctx.rank == 0:
        mixed = args.precision == "mixed"
        info, cfg = main["info"], main["cfg"]
        workload = WORKLOADS.get(args.config, args.config)
        if args.config == "c5":
            workload += f"; n = {ctx.world}: w = {cfg['shell'][0]}/1024, {main['n_leaf_dofs']:,} DoFs"
        out = {"metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": ctx.world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
               "scaling": "weak" if args.config == "c5" else "strong", "vs_baseline": None,
               "dtype": "f32" if mixed else "f64", "data": "synthetic",
               "config": {"workload": workload, "config": args.config,
                          "precision": "fp32 V-cycle in fp64 CG" if mixed else "fp64",
                          "n_leaf_dofs": main["n_leaf_dofs"], "n_free_dofs": main["n_free_dofs"],
                          "levels": main["levels"], "level_dofs": info["level_dofs"], "k": cfg["k"],
                          "dim": cfg["dim"], "cheb_degree": args.cheb_degree, "global_batch": 1,
                          "l2": "inputs larger than L2 (MG-layout vectors %.0f MB each > 126 MB)"
                                % main["mg_vector_mb"],
                          "parallelism": "single GPU" if ctx.world == 1 else
                          f"{ctx.world} ranks, SFC partition ({args.partition}), levels <= {args.coarse_cells} cells "
                          f"on rank 0, {args.transport} ghost exchange",
                          "partition": args.partition, "partition_eta": main["partition_eta"],
                          "ghost_children_ratio": main["ghost_children_ratio"], "setup_s": main["setup_s"],
                          "setup": main["setup"], "grandfamily_patches": sum(info["level_gf"]),
                          "r1_rows_finest": info["level_r1"][-1]},
               "roofline": main["roofline"], "apply_plain": main["apply_plain"], "kernels": main["kernels"],
               "cpu_baseline": cpu, "e2e": main["e2e"], "gpu_launches": main["gpu_launches"],
               "launches_per_vcycle": main["launches_per_vcycle"], "clocks": main["clocks"], "cg": main["cg"]}
        if sec is not None:
            out["secondary"] = {sec["config"]: {
                "workload": WORKLOADS.get(sec["config"], sec["config"]), "value": sec["value"], "unit": UNIT,
                "ms_per_step": sec["ms_per_step"], "n_leaf_dofs": sec["n_leaf_dofs"], "levels": sec["levels"],
                "roofline": sec["roofline"], "apply_plain": sec["apply_plain"], "kernels": sec["kernels"][:6],
                "gpu_launches": sec["gpu_launches"], "launches_per_vcycle": sec["launches_per_vcycle"],
                "clocks": sec["clocks"], "cg": sec["cg"], "partition_eta": sec["partition_eta"],
                "setup_s": sec["setup_s"]}}
        print(json.dumps(out), flush=True)
    ctx.close()


def dry_run_rank(args, rank, world):
    """One rank's host-only rank-local setup (no GPU, no communication): time and
    peak host RSS, as a dict."""
    import resource
    import paper_1904_03317_b200 as G
    from gmg_inputs import config, config_c5
    cfg = config_c5(world) if args.config == "c5" else config(args.config)
    t0 = time.time()
    f = G.gmg_forest_generate(G.recipe_from_config(cfg))
    t_forest = time.time() - t0
    part = G.gmg_partition(f, world, mode=args.partition, coarse_cells=args.coarse_cells if world > 1 else 0)
    t_part = time.time() - t0 - t_forest
    h = G.gmg_setup(f, part, k=cfg["k"], rank=rank, host_only=True, rank_local=True)
    t_setup = time.time() - t0
    info = h.info()
    out = {"rank": rank, "setup_s": round(t_setup, 1), "forest_s": round(t_forest, 1),
           "partition_s": round(t_part, 1), "topology_s": round(t_setup - t_forest - t_part, 1),
           "max_rss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 2),
           "owned_leaf_dofs": info["n_owned"],
           "owned_level_dofs": [int(h.local_level(l)["owned_key"].size) for l in range(info["n_levels"])],
           "ghost_level_dofs": [int(h.local_level(l)["ghost_key"].size) for l in range(info["n_levels"])]}
    if rank == 0:
        m = part.model()
        out.update(n_leaves=f.info()["n_leaves"], levels=info["n_levels"], partition_eta=m["eta"])
    return out


def dry_run(args):
    """--dry-run: the N-rank setup of a config on the host only.  Every rank's
    rank-local setup (the part of the hierarchy it would hold) is built in its own
    process -- at most --dry-run-parallel at a time, since ranks need no
    communication for it -- and reports setup time and peak host RSS; one JSON
    line (not a bench line).  E.g. `python bench.py --gpus 8 --config c5 --dry-run`
    shows that config 5 at 8 x 125M DoFs sets up within the host's RAM."""
    world = args.gpus
    if os.environ.get("GMG_DRY_RANK") is not None:
        print(json.dumps(dry_run_rank(args, int(os.environ["GMG_DRY_RANK"]), world)), flush=True)
        return
    procs, results = [], []
    pending = list(range(world))
    while pending or procs:
        while pending and len(procs) < max(1, args.dry_run_parallel):
            r = pending.pop(0)
            env = dict(os.environ, GMG_DRY_RANK=str(r))
            env.pop("WORLD_SIZE", None)
            procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                          stdout=subprocess.PIPE, text=True))
        p0 = procs.pop(0)
        out, _ = p0.communicate()
        if p0.returncode != 0:
            raise SystemExit(f"dry-run rank failed: rc {p0.returncode}")
        results.append(json.loads(out.strip().splitlines()[-1]))
    results.sort(key=lambda d: d["rank"])
    head = {k: results[0].pop(k) for k in ("n_leaves", "levels", "partition_eta")}
    print(json.dumps({"dry_run": True, "config": args.config, "n_ranks": world, **head,
                      "max_rss_gb_per_rank": max(r["max_rss_gb"] for r in results),
                      "max_setup_s": max(r["setup_s"] for r in results), "ranks": results}), flush=True)


def relaunch(args):
    """--gpus N > 1 outside torchrun: start N ranks with torch.distributed.run."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--secondary", default="c3", help="a second config measured in the same run, or 'none'")
    ap.add_argument("--cheb-degree", type=int, default=4)
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="NCCL (one GPU per rank) or host shared memory (any number of ranks per GPU; "
                         "a correctness path, not a performance one)")
    ap.add_argument("--partition", default="first_child", choices=["first_child", "per_level"],
                    help="level ownership: first-child rule (P:604, default) or per-level SFC balance (P:597)")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "mixed"],
                    help="fp64 V-cycle (default, BASELINE) or fp32 V-cycle inside the fp64 CG (P:897)")
    ap.add_argument("--coarse-cells", type=int, default=4096,
                    help="N > 1: levels with at most this many cells are gathered on rank 0 (0 = off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="cudaProfilerStart/Stop around one V-cycle of the headline config (ncu launch lists)")
    ap.add_argument("--dry-run", action="store_true",
                    help="host-only rank-local setup of every rank, reports time and host RSS (no GPU)")
    ap.add_argument("--dry-run-parallel", type=int, default=2, help="--dry-run: ranks set up concurrently")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return 0
    if args.dry_run:
        dry_run(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
