"""Benchmark of the recycled shifted solver hot path (arXiv 2306.15049) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C4] [--step outer|nested]

Workload (BASELINE.json): the largest single-GPU configuration C4 -- 1024 x 1024 image,
15 x 15 Gaussian PSF, 128 shifts gamma in [1e-6, 1e2], n_c = 80, |J| = 12, tau = 1e-4,
CG tol 1e-8 -- which is also north_star's 1 -> 8 GPU shift-sharding configuration.

A "step" (default --step outer) is one complete outer IRN step of C4 at k = 1 from a
frozen, device-resident snapshot of the state after outer step 0 (W_1, X^(0), G^(0),
V_i1; built once, untimed): stabilize [V_i1, X^(0)] (Alg. 1), anchoring + Grams, the
principal guesses of all 128 shifts (eq:orthupdate), the two group Ritz blocks (Alg. 2/4),
the carried corrections and their images, the batched deflated CG of all 128 shifts to
relres 1e-8 (every status must be CONVERGED), the L-curve corner and the IRN weights
of x*. Every step repeats identical work. --step nested times the whole nested solve
(K_out outer steps from W_0 = I) instead; the default run also reports one full
nested solve of the config (`nested_solve_s`) measured after the timed steps.

Metric value = A_gamma applies per second over the whole job (the paper's cost unit,
P:821-826; method accounting: CG iterations, true-residual confirmations, r_p, g-hat
images and anchoring applies). N GPUs (torchrun): the same problem, its shifts sharded
across the ranks (strong scaling); time = max over ranks.

Timing: CUDA events on the launching stream around each step, W untimed warm-up steps,
L2 (126 MB) flushed between steps by a 256 MB write outside the events; the working set
(~15 GB) is far larger than L2 anyway. One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import platform
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
CONVERGED = (0, 3)    # RSK_CG_CONVERGED, RSK_CG_DEFL_DROPPED (converged on a reduced space)


def _peaks():
    """HBM copy bandwidth (driver-measured MEASURED_PEAKS.json) and the FP64 DMMA /
    DFMA peaks measured on this pool's B200s (profiles/fp64_peak.json)."""
    out = {"hbm_gbs": 6650.0, "hbm_src": "fallback", "fp64_tflops": 37.0, "fp64_src": "nominal"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            out["hbm_gbs"] = float(json.load(f)["hbm_gbs"]); out["hbm_src"] = "measured"
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            p = json.load(f)
        out["fp64_tflops"] = float(p["dmma_tflops"]); out["fp64_src"] = "measured (profiles/fp64_peak.json)"
    except Exception:
        pass
    return out


def _cpu_desc():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return model, os.cpu_count() or 1


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
_OW = {}


def _oracle_init(cfg_name):
    """Worker set-up (once per process): the config's operator and right-hand side."""
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    from oracle import operators as ops
    from oracle import pipeline as opipe
    cfg = S.CONFIGS[cfg_name]
    inputs = S.make_inputs(cfg)
    h = opipe.operator_of(cfg, inputs)
    d, b = ops.make_data(h, inputs["x_true"], inputs["xi"], cfg.noise)
    _OW.update(cfg=cfg, h=h, b=b.ravel(), gamma=inputs["gamma"], w=ops.identity_weights(cfg.n))


def _oracle_worker(args):
    """One host core: the oracle as it stands (numpy fp64, one thread) running plain CG
    (O4 with U = empty, x_0 = 0, W_0 = I -- the seed-solve form of the same operator) at
    shift gamma_l for about `budget_s` seconds. Returns (applies, seconds)."""
    l, budget_s = args
    from oracle import defcg as dcg
    from oracle import operators as ops
    cfg, h, b = _OW["cfg"], _OW["h"], _OW["b"]
    wx, wy = _OW["w"]
    n = cfg.n
    g = float(_OW["gamma"][l])
    A = lambda v: ops.apply_shifted(h, wx, wy, g, v.reshape(n, n)).ravel()
    t0 = time.perf_counter()
    dcg.defcg(A, b, tol=1e-300, maxit=1)
    per = max(time.perf_counter() - t0, 1e-4) / 2.0
    its = max(1, int(budget_s / per))
    t0 = time.perf_counter()
    r = dcg.defcg(A, b, tol=1e-300, maxit=its)
    return r.applies, time.perf_counter() - t0


class OraclePool:
    """The oracle, untuned, on ALL host cores: one process per core (spawned once), each a
    plain CG of the config's operator at a different shift of the ladder."""

    def __init__(self, cfg, cores=None):
        self.model, ncpu = _cpu_desc()
        self.cores = cores or ncpu
        self.cfg = cfg
        self.ls = [int(round(i * (cfg.M - 1) / max(self.cores - 1, 1))) for i in range(self.cores)]
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_oracle_init, initargs=(cfg.name,))

    def sample(self, budget_s):
        """Returns (applies/s, cores, description) of one bounded sample."""
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_worker, [(l, budget_s) for l in self.ls], chunksize=1)
        wall = time.perf_counter() - t0
        ap = sum(a for a, _ in res)
        busy = max(t for _, t in res)
        cfg = self.cfg
        return ap / busy, self.cores, (f"oracle (numpy fp64) plain CG on {cfg.name} (n={cfg.n}, {2*cfg.r+1}x{2*cfg.r+1} "
                                       f"PSF), one shift per core over the ladder, {ap} applies in {busy:.1f} s on "
                                       f"{self.cores} cores ({self.model}); wall {wall:.1f} s")

    def close(self):
        self.pool.close()
        self.pool.join()


def oracle_sample(cfg, budget_s, cores=None):
    p = OraclePool(cfg, cores)
    try:
        return p.sample(budget_s)
    finally:
        p.close()


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    pool = OraclePool(cfg)
    for _ in range(max(1, args.warmup)):
        pool.sample(1.0)                        # warm-up (process start, imports, set-up)
    vals = []
    desc = cores = None
    t_total = time.perf_counter()
    for _ in range(args.steps):
        v, cores, desc = pool.sample(args.ref_budget)
        vals.append(v)
    t_total = time.perf_counter() - t_total
    pool.close()
    v = float(np.mean(vals))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": cfg.name, "n": cfg.n, "shifts": cfg.M, "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU leg
def alg_bytes_per_shift_iteration_px(J, S_gpu, n_grp):
    """one Def-CG shift-iteration moves 80 B/px of per-shift vectors (x,
    r, p read + write; w write + read; g-hat and its image) plus the shared group blocks
    W, AW, EW (24 |J| B/px per group present) and the weights (16 B/px), amortised over
    the S shifts of the batch on this GPU."""
    return 80.0 + (n_grp * 24.0 * J + 16.0) / max(S_gpu, 1)


def run_ours(args, cfg, rank, world):
    import torch
    import torch.distributed as dist
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200 import shard
    from paper_2306_15049_b200.pipeline import GpuSolver

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("RSK_BENCH_SAME_GPU"):   # test hook: every rank on cuda:0 (gloo)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = L.load()
    stream = torch.cuda.current_stream(dev)
    inputs = S.make_inputs(cfg)
    D = shard.Dist(world > 1)
    sol = GpuSolver(cfg, inputs["psf"], inputs["gamma"], device=local, check_every=args.check_every, dist=D)
    x_true = torch.from_numpy(inputs["x_true"]).to(dev)
    xi = torch.from_numpy(inputs["xi"]).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    nested = args.step == "nested"
    f = dict(dtype=torch.float64, device=dev)
    wnx = torch.empty(cfg.N, **f)
    wny = torch.empty(cfg.N, **f)

    # ---- the frozen snapshot after outer step 0 (untimed)
    t_setup = time.perf_counter()
    sol.set_data(x_true, xi)
    sol.reset_weights()
    snap = None
    if not nested:
        o0, st0 = sol.outer_step(0, {})
        sol.next_weights(st0["xstar"])
        st0["W_prev"] = sol.w_prev
        W1 = (sol.wx.clone(), sol.wy.clone())
        snap = dict(st0)
    t_setup = time.perf_counter() - t_setup

    def step():
        if nested:
            sol.set_data(x_true, xi)
            return sol.run()
        sol.h.set_weights(W1[0], W1[1], stream=sol.stream)
        o, st = sol.outer_step(1, snap)
        sol.h.irn_weights(st["xstar"], cfg.tau, wnx, wny, stream=sol.stream)   # H1: W_2 from x*
        sol.last_state = st
        return [o]

    def count(outs):
        ap = sum(int(o.applies.sum()) + o.overhead_applies for o in outs)
        sv = sum(int(o.applies.size) for o in outs)
        its = sum(int(o.iters.sum()) for o in outs)
        conv = sum(int(np.isin(o.status, CONVERGED).sum()) for o in outs)
        return ap, sv, its, conv

    for _ in range(args.warmup):
        outs = step()
    torch.cuda.synchronize(dev)
    D.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    tot_ap = tot_sv = tot_it = tot_conv = 0
    loop_ms = loop_its = 0.0
    loop_launches = 0
    kinds = set()
    l0 = lib.rsk_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))                       # L2 flush between timed steps (256 MB > 126 MB L2)
            ev[i][0].record(stream)
            outs = step()
            ev[i][1].record(stream)
            ap, sv, it, conv = count(outs)
            tot_ap += ap; tot_sv += sv; tot_it += it; tot_conv += conv
            for o in outs:
                if o.prof is not None:
                    loop_ms += float(o.prof[5]); loop_its += float(o.prof[6]); kinds.add(int(o.prof[7]))
                    loop_launches += int(np.ceil(float(o.prof[2]) / 512.0))   # 512 lockstep iterations per launch
        torch.cuda.synchronize(dev)
    launches = lib.rsk_launch_count() - l0
    ms = sum(a.elapsed_time(b) for a, b in ev)
    # the per-shift arrays of every StepOut are all-gathered (global), so the counts are
    # the whole job's; the device-loop time and shift-iterations are this rank's
    mine = torch.tensor([ms, loop_ms, loop_its], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mine[:1], op=dist.ReduceOp.MAX)
    ms = float(mine[0])
    value = tot_ap / (ms / 1e3)
    solves = tot_sv / (ms / 1e3)
    last = outs
    all_conv = tot_conv == tot_sv
    if not all_conv and rank == 0:
        sys.stderr.write(f"bench: {tot_sv - tot_conv} of {tot_sv} solves not CONVERGED\n")

    # ---- e2e through the public API with host buffers (pinned): every step copies its
    # inputs host -> device (the snapshot state, or x_true / xi for the nested solve) and
    # its solutions X device -> host inside the timed region
    e2e_steps = max(1, min(args.steps, 3))
    if nested:
        h_in = [torch.from_numpy(inputs["x_true"]).pin_memory(), torch.from_numpy(inputs["xi"]).pin_memory()]
        d_in = [x_true, xi]
    else:
        # (ranks other than 0 hold no V_i1: rank 0 builds the principal space, shard.py)
        d_in = [t for t in (snap["X_prev"], snap["G_prev"], snap["V_i1"], W1[0], W1[1]) if t is not None]
        h_in = [t.cpu().pin_memory() for t in d_in]
    res_h = torch.empty(cfg.M, cfg.N, dtype=torch.float64).pin_memory()
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e2e_steps)]
    e_ap = 0
    for i in range(e2e_steps):
        flush.fill_(float(i))
        ee[i][0].record(stream)
        for hd, dd in zip(h_in, d_in):
            dd.copy_(hd, non_blocking=True)
        outs_e = step()
        Xres = sol.final["X_prev"] if nested else sol.last_state["X_prev"]
        res_h.copy_(Xres, non_blocking=True)
        ee[i][1].record(stream)
        e_ap += count(outs_e)[0]
    torch.cuda.synchronize(dev)
    ems = sum(a.elapsed_time(b) for a, b in ee)
    if world > 1:
        t = torch.tensor([ems], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    e2e = {"value": e_ap / (ems / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(sum(t.numel() * t.element_size() for t in h_in)),
           "d2h_bytes_per_step": int(cfg.M * cfg.N * 8)}

    # ---- roofline of the dominant kernel: the device CG loop (persistent lockstep kernel
    # for images beyond L2, cluster-per-shift kernel otherwise), timed with CUDA events on
    # its launching stream inside librsk (StepOut.prof[5..6]) over the timed steps
    pk = _peaks()
    S_gpu = max(1, int(np.ceil(cfg.M / world)))
    per_px = alg_bytes_per_shift_iteration_px(cfg.J, S_gpu, 2)
    alg_bytes = per_px * cfg.N * loop_its
    achieved = alg_bytes / (loop_ms / 1e3) / 1e9 if loop_ms > 0 else None
    kind = max(kinds) if kinds else 0
    n_launch_loop = 0
    # DRAM traffic of the loop kernel per launch: the DRAM bytes per ms of the committed
    # ncu --set full capture of one k = 1 launch (profiles/r2/cg_loop_traffic.json) x this
    # run's mean launch duration
    traffic = None
    tf = os.path.join(ROOT, "profiles", "r2", "cg_loop_traffic.json")
    if os.path.exists(tf) and loop_launches:
        with open(tf) as fh:
            tr = json.load(fh)
        if tr.get("workload") == cfg.name and world == 1:
            traffic = tr["dram_bytes_per_ms"] * loop_ms / loop_launches
    # standalone fused apply over the full batch (all M shifts): 10 back-to-back launches
    # between two events, best of 3; FP64 work (16 r + 20) flop/px
    X = torch.randn(cfg.M, cfg.N, **f)
    Y = torch.empty_like(X)
    best = 1e9
    for _ in range(3):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(10):
            sol.h.apply_shifted(X, Y, gamma=sol.gam_dev)
        a1.record(stream)
        torch.cuda.synchronize(dev)
        best = min(best, a0.elapsed_time(a1) / 10)
    del X, Y
    sa_bytes = 16.0 * cfg.M * cfg.N + 16.0 * cfg.N
    sa_flop = (16.0 * cfg.r + 20.0) * cfg.N * cfg.M
    tf_ach = sa_flop / (best / 1e3) / 1e12
    apply_roof = {"bound": "fp64" if (16 * cfg.r + 20) / 16.0 > pk["fp64_tflops"] * 1e3 / pk["hbm_gbs"] else "hbm",
                  "ms": best, "applies_per_s": cfg.M / (best / 1e3),
                  "achieved_tflops": tf_ach, "peak_tflops": pk["fp64_tflops"], "frac_fp64": tf_ach / pk["fp64_tflops"],
                  "achieved_gbs": sa_bytes / (best / 1e3) / 1e9, "peak_gbs": pk["hbm_gbs"],
                  "frac_hbm": sa_bytes / (best / 1e3) / 1e9 / pk["hbm_gbs"],
                  "alg_flop_per_px": 16 * cfg.r + 20, "alg_bytes_per_px": 16.0 + 16.0 / cfg.M,
                  "peak_src": pk["fp64_src"]}

    # ---- one full nested solve of the config (K_out outer steps), if it fits the budget
    nested_s = None
    outs_n = None
    if not nested and not args.no_nested and (ms / args.steps) * cfg.K_out / 1e3 < args.nested_budget:
        torch.cuda.synchronize(dev)
        D.barrier()
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0.record(stream)
        sol.set_data(x_true, xi)
        outs_n = sol.run()
        n1.record(stream)
        torch.cuda.synchronize(dev)
        nested_s = n0.elapsed_time(n1) / 1e3
        if world > 1:
            t = torch.tensor([nested_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            nested_s = float(t.item())
        nested_info = {"s": nested_s, "outer_steps": len(outs_n),
                       "applies": int(sum(int(o.applies.sum()) + o.overhead_applies for o in outs_n)),
                       "cg_iterations": [int(o.iters.sum()) for o in outs_n],
                       "lstar": [int(o.lstar) for o in outs_n],
                       "converged": f"{sum(int(np.isin(o.status, CONVERGED).sum()) for o in outs_n)}"
                                    f"/{sum(int(o.status.size) for o in outs_n)}"}
    else:
        nested_info = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, desc = oracle_sample(cfg, args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0 and args.report:
        from paper_2306_15049_b200.pipeline import report_rows
        rows = report_rows(outs_n if nested_info else last, inputs["gamma"])
        import csv
        with open(args.report, "w", newline="") as fh:
            wr = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
            wr.writeheader()
            wr.writerows(rows)
    if rank == 0:
        o = last[-1]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "N": cfg.N, "shifts": cfg.M,
                       "step": ("nested solve, K_out outer steps" if nested else
                                "outer step k=1 from a frozen snapshot after k=0"),
                       "inner": cfg.inner, "local": cfg.local, "weight_rule": cfg.weight_rule,
                       "principal": cfg.principal, "operator": cfg.operator, "outer_steps": cfg.K_out,
                       "n_c": cfg.n_c, "J": cfg.J, "psf": f"{2*cfg.r+1}x{2*cfg.r+1}", "tau": cfg.tau,
                       "tol": cfg.tol, "maxit": cfg.maxit,
                       "l2": "flushed between steps (256 MB write); working set > L2",
                       "parallelism": (f"shift-sharded x{world} (NCCL): one principal-space exchange "
                                       f"per outer step, no per-iteration communication") if world > 1 else "single"},
            "solves_per_s": solves,
            "applies_per_step": tot_ap / args.steps, "cg_iterations_per_step": tot_it / args.steps,
            "converged": f"{tot_conv}/{tot_sv}", "all_converged": bool(all_conv),
            "lstar": [int(x.lstar) for x in last],
            "iters_max": int(max(int(x.iters.max()) for x in last)),
            "setup_s": t_setup,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm",
                         "kernel": {1: "cg_cluster_kernel (cluster-per-shift deflated CG loop)",
                                    2: "cg_persist_kernel (tiled persistent lockstep deflated CG loop)",
                                    3: "cg_stream_kernel (streaming persistent lockstep deflated CG loop)"}.get(kind, "host-polled loop"),
                         "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": (achieved / pk["hbm_gbs"]) if achieved else None, "traffic": traffic,
                         "peak_src": pk["hbm_src"],
                         "alg_bytes_per_shift_iteration_px": per_px,
                         "alg_formula": "80 + (n_grp*24*J + 16)/S, S = shifts per GPU, n_grp = 2 (SURVEY 8(d) d2)",
                         "shift_iterations": loop_its, "kernel_ms": loop_ms, "N": cfg.N,
                         "launches": loop_launches,
                         "alg_bytes_per_launch": (alg_bytes / loop_launches) if loop_launches else None,
                         "kernel_ms_share": loop_ms / max(ms, 1e-9)},
            "apply_roofline": apply_roof,
            "nested_solve": nested_info,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def run_slab(args, cfg, rank, world):
    """C5 across G GPUs as row slabs: every rank holds its rows (+ 2r halo)
    of all 16 shifts; halo exchange and the all-reduced dot products over NCCL
    (slab.DistComm). A step = outer step k = 0 of the nested solve (seed solves, Ritz,
    stabilize, anchoring, guesses, group blocks, batched deflated CG, L-curve)."""
    import torch
    import torch.distributed as dist
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.slab import DistComm, SlabGpuSolver, SlabPlan
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("RSK_BENCH_SAME_GPU"):   # test hook: every rank on cuda:0 (gloo)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = L.load()
    inputs = S.make_inputs(cfg)
    plan = SlabPlan(cfg.n, cfg.n, cfg.r, world)
    sol = SlabGpuSolver(cfg, inputs["psf"], inputs["gamma"], plan, rank, DistComm(plan, rank), device=local)
    x_true = torch.from_numpy(inputs["x_true"]).to(dev)
    xi = torch.from_numpy(inputs["xi"]).to(dev)

    def step():
        sol.set_data(x_true, xi)
        sol.reset_weights()
        o, _ = sol.outer_step(0, {})
        return o

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    stream = torch.cuda.current_stream(dev)
    ms = 0.0
    ap = sv = conv = 0
    l0 = lib.rsk_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            o = step()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms += e0.elapsed_time(e1)
            ap += int(o.applies.sum()) + o.overhead_applies
            sv += int(o.applies.size)
            conv += int(np.isin(o.status, CONVERGED).sum())
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0 and args.report:
        from paper_2306_15049_b200.pipeline import report_rows
        import csv
        rows = report_rows([o], inputs["gamma"])
        with open(args.report, "w", newline="") as fh:
            wr = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
            wr.writeheader()
            wr.writerows(rows)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": ap / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "N": cfg.N, "shifts": cfg.M, "step": "outer step k=0",
                       "parallelism": f"row slabs x{world} (NCCL halo exchange + all-reduced dots)",
                       "l2": "working set > L2"},
            "solves_per_s": sv / (ms / 1e3), "converged": f"{conv}/{sv}",
            "gpu_launches": int(lib.rsk_launch_count() - l0), "clocks": clk.summary(),
        }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--step", default="outer", choices=["outer", "nested"])
    ap.add_argument("--check-every", type=int, default=8)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=5.0)
    ap.add_argument("--nested-budget", type=float, default=300.0)
    ap.add_argument("--no-nested", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--report", default=None, help="CSV of the per-(k, l) accounting of the last step / nested solve")
    ap.add_argument("--slab", action="store_true", help="row slabs across the ranks (default for C5 at N > 1)")
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
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    # --slab at one rank runs the row-slab solver on a single slab (the N = 1 point of the
    # slab scaling curve; a process group of one)
    slab = (world > 1 and cfg.name == "C5") or args.slab
    if world > 1 or slab:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group(os.environ.get("RSK_BENCH_BACKEND", "nccl"), rank=rank, world_size=world)
    if slab:
        run_slab(args, cfg, rank, world)
    else:
        run_ours(args, cfg, rank, world)
    if world > 1 or slab:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
