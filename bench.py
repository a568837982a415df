"""Benchmark of the recycled shifted solver hot path (arXiv 2306.15049) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

A "step" is one pass of the whole hot path over one batch of synthetic input:
the complete nested solve of a BASELINE.json configuration (K_out outer IRN
steps x M shifts: data d, b; seed solves + Ritz; stabilize; anchoring + Grams;
principal guesses; group Ritz blocks; carried corrections; batched deflated CG;
L-curve; IRN weights). Default workload: configs[1] = C2 (256x256, 32 shifts,
5 outer steps). Metric value = fused (A + gamma E_k) applies per second over the
whole job (method accounting: every A_gamma apply, seeds/Ritz/anchoring included).

Timing: CUDA events on the launching stream around each step, L2 flushed between
steps (outside the events), W untimed warm-up steps, max over ranks.
One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import rsk_synth as S  # noqa: E402

METRIC = "fused (A+γE_k)x applies/s & shifted solves/s; HBM GB/s vs peak, 1-8 GPU"
UNIT = "applies/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU oracle leg
def oracle_sample(cfg, inputs, budget_s=12.0):
    """The oracle as it stands (numpy fp64, single thread) on a bounded sample of the
    same workload: plain CG at gamma_i1 from x = 0 on the config's own b, W_0 = I --
    the seed solve that opens the nested solve -- stopped after `budget_s` seconds.
    Returns applies/s (same unit as the GPU metric)."""
    from oracle import defcg as dcg
    from oracle import operators as ops
    from oracle import pipeline as opipe
    n = cfg.n
    h = opipe.operator_of(cfg, inputs)   # the PSF, or the CT matrix (C6)
    d, b = ops.make_data(h, inputs["x_true"], inputs["xi"], cfg.noise)
    wx, wy = ops.identity_weights(n)
    g = float(inputs["gamma"][0])   # gamma_i1, i1 = 1
    A = lambda v: ops.apply_shifted(h, wx, wy, g, v.reshape(n, n)).ravel()
    # time a few iterations to size the sample to the budget
    t0 = time.perf_counter()
    dcg.defcg(A, b.ravel(), tol=1e-300, maxit=2)
    per = max((time.perf_counter() - t0) / 4.0, 1e-4)
    its = max(2, int(budget_s / per))
    t0 = time.perf_counter()
    r = dcg.defcg(A, b.ravel(), tol=1e-300, maxit=its)
    dt = time.perf_counter() - t0
    return r.applies / dt, f"oracle plain CG at gamma_i1 on {cfg.name} (n={n}), {r.applies} applies in {dt:.1f}s"


def run_reference(args, cfg, inputs, rank, world):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    if rank != 0:
        return
    vals = []
    for _ in range(args.warmup):
        oracle_sample(cfg, inputs, budget_s=1.0)
    t_total = time.perf_counter()
    for _ in range(args.steps):
        v, desc = oracle_sample(cfg, inputs, budget_s=args.ref_budget)
        vals.append(v)
    t_total = time.perf_counter() - t_total
    v = float(np.mean(vals))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": cfg.name, "n": cfg.n, "shifts": cfg.M,
                                        "outer_steps": cfg.K_out, "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU leg
def run_ours(args, cfg, inputs, rank, world):
    import torch
    import torch.distributed as dist
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.pipeline import GpuSolver

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("RSK_BENCH_SAME_GPU"):   # test hook: every rank on cuda:0 (gloo)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = L.load()
    stream = torch.cuda.current_stream(dev)
    from paper_2306_15049_b200 import shard
    sol = GpuSolver(cfg, inputs["psf"], inputs["gamma"], device=local, check_every=args.check_every,
                    dist=shard.Dist(world > 1))
    x_true = torch.from_numpy(inputs["x_true"]).to(dev)
    xi = torch.from_numpy(inputs["xi"]).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def step():
        sol.set_data(x_true, xi)
        outs = sol.run()
        return outs

    def count(outs):
        ap = sum(int(o.applies.sum()) + o.overhead_applies for o in outs)
        sv = sum(int(o.applies.size) for o in outs)
        its = sum(int(o.iters.sum()) for o in outs)
        return ap, sv, its

    for _ in range(args.warmup):
        outs = step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    tot_ap = tot_sv = tot_it = 0
    l0 = lib.rsk_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))                       # L2 flush between timed steps (256 MB > 126 MB L2)
            ev[i][0].record(stream)
            outs = step()
            ev[i][1].record(stream)
            ap, sv, it = count(outs)
            tot_ap += ap; tot_sv += sv; tot_it += it
        torch.cuda.synchronize(dev)
    launches = lib.rsk_launch_count() - l0
    ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # the per-shift arrays of every StepOut are already global (all-gathered), so the
    # counts are the whole job's, not this rank's
    tot_ap_all, tot_sv_all = tot_ap, tot_sv
    value = tot_ap_all / (ms / 1e3)
    solves = tot_sv_all / (ms / 1e3)
    last = outs

    # ---- e2e through the public API with host buffers (pinned), copies inside the region
    xt_h = torch.from_numpy(inputs["x_true"]).pin_memory()
    xi_h = torch.from_numpy(inputs["xi"]).pin_memory()
    res_h = torch.empty(cfg.M, cfg.N, dtype=torch.float64).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e2e_steps)]
    e_ap = 0
    for i in range(e2e_steps):
        flush.fill_(float(i))
        ee[i][0].record(stream)
        x_true.copy_(xt_h, non_blocking=True)
        xi.copy_(xi_h, non_blocking=True)
        outs = step()
        res_h.copy_(sol.final["X_prev"], non_blocking=True)
        ee[i][1].record(stream)
        e_ap += count(outs)[0]
    torch.cuda.synchronize(dev)
    ems = sum(a.elapsed_time(b) for a, b in ee)
    if world > 1:
        t = torch.tensor([ems], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    e2e = {"value": e_ap / (ems / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": 2 * cfg.N * 8, "d2h_bytes_per_step": cfg.M * cfg.N * 8}

    # ---- roofline of the dominant kernel: the device-side CG loop (cluster-per-shift
    # kernel for L2-resident images, persistent lockstep kernel otherwise), timed live with
    # CUDA events on its launching stream inside librsk over the timed steps (ms_loop[5..7]).
    prof_all = [o.prof for o in last]
    dl_ms = float(sum(p[5] for p in prof_all))
    dl_its = float(sum(p[6] for p in prof_all))
    kind = int(max(p[7] for p in prof_all)) if prof_all else 0
    J = cfg.J
    # algorithmic bytes per shift-iteration and pixel: apply p, w, W_k (32);
    # update w, r, r', ZGhat, Z = AW + gamma EW (32 + 8 J); combine p, x, r, ghat, p', x',
    # W (48 + 8 J). Lockstep batches share AW, EW, W (24 J) over a group's shifts.
    per_px = (32 + 32 + 48 + 16 * J) if kind == 1 else (32 + 32 + 48 + 24 * J / max(1.0, cfg.M / 2))
    alg_bytes = per_px * cfg.N * dl_its
    achieved = alg_bytes / (dl_ms / 1e3) / 1e9 if dl_ms > 0 else None
    peak, peak_src = _peaks()
    step_ms_last = ms / args.steps
    # DRAM traffic of the dominant kernel per launch: bytes per shift-iteration from the
    # committed ncu --set full capture (profiles/r1/cg_cluster_traffic.json) times this
    # step's shift-iterations per launch (one launch per outer step)
    traffic = None
    nl = sum(1 for p in prof_all if p[6] > 0)
    tf = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1", "cg_cluster_traffic.json")
    if kind == 1 and nl and os.path.exists(tf) and cfg.name == "C2":
        with open(tf) as f:
            traffic = json.load(f)["dram_bytes_per_shift_iteration"] * dl_its / nl
    # standalone fused apply over the full batch (all M shifts): 20 back-to-back launches
    # between two events (no host gaps inside), best of 3
    X = torch.randn(cfg.M, cfg.N, dtype=torch.float64, device=dev)
    Y = torch.empty_like(X)
    best = 1e9
    for _ in range(4):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(20):
            sol.h.apply_shifted(X, Y, gamma=sol.gam_dev)
        a1.record(stream)
        torch.cuda.synchronize(dev)
        best = min(best, a0.elapsed_time(a1) / 20)
    sa_bytes = 16.0 * cfg.M * cfg.N + 16.0 * cfg.N
    standalone = {"applies_per_s": cfg.M / (best / 1e3), "ms": best,
                  "gbs": sa_bytes / (best / 1e3) / 1e9, "frac_hbm": sa_bytes / (best / 1e3) / 1e9 / peak}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        v, desc = oracle_sample(cfg, inputs, budget_s=args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "N": cfg.N, "shifts": cfg.M,
                       "inner": cfg.inner, "local": cfg.local, "weight_rule": cfg.weight_rule,
                       "principal": cfg.principal, "operator": cfg.operator,
                       "outer_steps": cfg.K_out, "n_c": cfg.n_c, "J": cfg.J, "psf": f"{2*cfg.r+1}x{2*cfg.r+1}",
                       "tol": cfg.tol, "l2": "flushed between steps (256 MB write)",
                       "parallelism": (f"shift-sharded x{world} (NCCL): {cfg.ladder_base} shifts per GPU, "
                                       f"one principal-space exchange per outer step") if world > 1 else "single"},
            "solves_per_s": solves,
            "applies_per_step": tot_ap / args.steps, "cg_iterations_per_step": tot_it / args.steps,
            "lstar": [int(o.lstar) for o in last],
            "iters_per_outer_step": [int(o.iters.sum()) for o in last],
            "e2e": e2e,
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm",
                         "kernel": {1: "cg_cluster_kernel (cluster-per-shift deflated CG loop)",
                                    2: "cg_persist_kernel (persistent lockstep deflated CG loop)"}.get(kind, "host-polled loop"),
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_unit": "B per launch (ncu dram__bytes_read+write, L2-resident: far below"
                                         " the algorithmic bytes)",
                         "alg_bytes_per_launch": (alg_bytes / nl) if nl else None,
                         "peak_source": peak_src,
                         "kernel_ms_per_step": dl_ms, "kernel_ms_share": dl_ms / max(step_ms_last, 1e-9),
                         "shift_iterations_per_step": dl_its,
                         "alg_bytes_per_shift_iteration_px": per_px,
                         "working_set": "L2-resident (126 MB L2)" if cfg.N * cfg.M * 8 * 6 < 126e6 else "HBM"},
            "apply_standalone": standalone,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--check-every", type=int, default=8)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    # options of the nested solve (defaults = north_star's path; see README / DESIGN)
    ap.add_argument("--inner", default=None, choices=["cg", "minres"])
    ap.add_argument("--local", default=None, choices=["d3", "seq"])
    ap.add_argument("--rule", default=None, choices=["irn", "irn_iso", "gazzola"])
    ap.add_argument("--principal", default=None, choices=["g10", "vnew"])
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = S.CONFIGS[args.config]
    import dataclasses
    over = {k: v for k, v in (("inner", args.inner), ("local", args.local), ("weight_rule", args.rule),
                              ("principal", args.principal)) if v is not None}
    if cfg.operator == "ct":
        over.setdefault("inner", "minres")
    if over:
        cfg = dataclasses.replace(cfg, **over)
    inputs = S.make_inputs(cfg)
    if args.impl == "reference":
        run_reference(args, cfg, inputs, rank, world)
        return
    if world > 1:
        # weak scaling by shift (reading G39): the ladder is densified to
        # M = 32 N shifts over the same gamma range, 32 per GPU; the principal space keeps
        # the N = 1 sizes (every N-th previous solution in the k >= 1 raw block)
        cfg = dataclasses.replace(cfg, M=cfg.M * world, ladder_base=cfg.M)
        inputs = S.make_inputs(cfg)
        import torch.distributed as dist
        dist.init_process_group(os.environ.get("RSK_BENCH_BACKEND", "nccl"))
    run_ours(args, cfg, inputs, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
