"""Benchmark: spaND factorize + PCG solve on BASELINE config C4 (headline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C4] [--levels 15] [--no-cpu-baseline]

Workload (BASELINE.json configs[3]): 3D 64^3 high-contrast diffusion,
7-point finite volumes with harmonic faces, a piecewise constant on 8^3
blocks with log10 a ~ U(-3, 3) (seed 3), n = 262144, nested dissection to
15 levels, eps = 1e-2, second-order "second-full" scheme, skip_levels = 4,
b ~ N(0, 1) from the same generator, PCG to relative residual 1e-12.
Synthetic input built in-process (no dataset involved).

A STEP is one full pass of the hot path: factorize(A, hierarchy) on the
B200 followed by pcg(A, b, M) to 1e-12 (the hierarchy is the factorize
input, as in the reference API; it is built once, on the host, and timed
separately).  metric = algorithmic FP64 work of the step (F_elim +
F_scale + F_rrqr + 4 nnz_factor per apply + 2 nnz(A) per SpMV, formulas in
paper_2007_00789_b200/metrics.py) / step time, in GFLOP/s
(higher is better); the same formula prices the CPU oracle's step, so the
ratio is work-normalised even though the CPU runs a smaller sample.
  value : inputs resident in HBM (A's device CSR and block-scatter arrays
          cached on the device, b a device tensor, x left on the device);
  e2e   : the public API from host buffers (a fresh SparseSymMatrix and a
          NumPy b every step, x returned to the host): host->device copies
          of A and b and the device->host copy of x inside the timed region.
Timing: barrier + cuda.synchronize on both sides of the K timed steps,
CUDA events on the launching stream, max over ranks; L2 flushed (256 MiB
write) between steps; the factor (> 2 GB) exceeds L2 anyway.
N > 1: replicas only (the path does not shard): every rank
factors and solves its own copy; value = N * n / max-rank step time.

--impl reference: the CPU oracle port (oracle/spand_oracle.py, a bitwise
restatement of the reference spdkit, see tests/test_oracle_golden.py) on a
bounded sample of the same workload family, all host threads, rank 0 only.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = ("spaND factorize+PCG-solve FP64 throughput (algorithmic GFLOP/s: "
          "F_elim+F_scale+F_rrqr+apply+SpMV per step / step time)")
FP64_PEAK_TFLOPS = 36.5   # measured DFMA loop on this pool's B200, profiles/fp64_peak_r01.jsonl
FP64_DGEMM_TFLOPS = 35.5  # measured cuBLAS DGEMM (8192^3), same file
SAMPLE = {"grid": 24, "block": 8, "levels": 11, "seed": 3}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4")
    p.add_argument("--levels", type=int, default=None)
    p.add_argument("--eps", type=float, default=1e-2)
    p.add_argument("--scheme", default="second-full")
    p.add_argument("--tol", type=float, default=1e-12)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-near-kernel", action="store_true",
                   help="skip the near-kernel (extension) side measurement")
    return p.parse_args()


def dist_init(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (clocks + throttle reasons)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def reduce_max(v, dist, device):
    """Max of a per-rank scalar over all ranks (the step time of the job)."""
    if dist is None:
        return v
    import torch
    tv = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(tv, op=dist.ReduceOp.MAX)
    return float(tv.item())


def whole_job_rate(work_per_rank, world, ms_step):
    """Replicas: every rank does the same work; the job's rate is the work of
    all ranks over the slowest rank's step time."""
    return world * work_per_rank / (ms_step / 1000.0)


def problem(args):
    import paper_2007_00789_b200 as sp
    a, b, lv = sp.baseline_problem(args.config)
    return a, b, (args.levels or lv)


def sample_problem():
    """Bounded CPU sample of the C4 family: same generator and seeding
    convention on a 24^3 grid (3x3x3 blocks of 8^3 cells), levels 11.
    Built with the oracle's restatement of the generator (bitwise equal to
    the package's, tests/test_host.py) so the CPU legs never load the
    product."""
    from oracle import spand_oracle as orc
    g = SAMPLE["grid"]
    n, rp, ci, va, b = orc.fv_block_field_problem((g, g, g), SAMPLE["block"], 3.0,
                                                  SAMPLE["seed"])
    return (n, rp, ci, va), b, SAMPLE["levels"]


def _metrics():
    """paper_2007_00789_b200/metrics.py loaded by path (numpy only): the
    algorithmic-work formulas, without importing the product package."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "spand_metrics_standalone", os.path.join(HERE, "paper_2007_00789_b200", "metrics.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def cpu_run(csr, b, levels, eps, scheme, tol, threads):
    """One factorize + PCG of the CPU oracle (timed, hierarchy excluded).
    Returns (seconds, n_cg, algorithmic flops of the step)."""
    from threadpoolctl import threadpool_limits
    from oracle import spand_oracle as orc
    met = _metrics()
    n, rp, ci, va = csr
    cl = orc.nd_hierarchy(n, rp, ci, levels)
    with threadpool_limits(limits=threads, user_api="blas"):
        t0 = time.perf_counter()
        f = orc.factorize(n, rp, ci, va, cl, levels, eps, scheme, 4)
        mv = orc.csr_matvec(n, rp, ci, va)
        _, its, _, _, _, _ = orc.pcg(mv, b, f.apply_m, tol)
        dt = time.perf_counter() - t0
    panels = [(op.dofs.size, op.n_cols, len(op.pivots)) for op in f.ops if op.kind == "Q"]
    fl = met.factor_flops(f.ops, panels)["F_factor"] + met.solve_flops(
        f.nnz_factor, rp[-1], its + 1, its + 1)
    return dt, its, fl


def reference_full_config(args):
    """The reference's own run of the headline config (frozen by
    tests/golden/make_golden.py in the build container: unmodified spdkit,
    1 OpenBLAS thread) -- the only same-config CPU figure: the reference
    cannot finish a C4-L15 step inside a bench run."""
    tag = f"{args.config}_L{args.levels or 15}_e{args.eps:g}_{args.scheme}"
    path = os.path.join(HERE, "tests", "golden", tag + ".json")
    try:
        with open(path) as fh:
            rec = json.load(fh)
    except OSError:
        return None
    return {"factorize_s": rec["t_factor_s"], "solve_s": rec["t_solve_s"],
            "hierarchy_s": rec["t_hier_s"], "n_cg": rec["n_cg"],
            "step_s": rec["t_factor_s"] + rec["t_solve_s"],
            "blas_threads": rec.get("blas_threads"), "versions": rec.get("versions"),
            "source": f"tests/golden/{tag}.json: unmodified reference spdkit "
                      "factorize + pcg on this workload in the build container "
                      "(make_golden.py), not timed in this run"}


def run_reference(args, rank):
    if rank != 0:
        return
    csr, b, lv = sample_problem()
    # all host cores are available; multi-threaded BLAS on the reference's
    # many small blocks can be slower than one thread, so the first warm-up
    # step tries both and the timed steps use the faster setting
    allc = os.cpu_count() or 1
    threads = allc
    if allc > 1:
        t1 = cpu_run(csr, b, lv, args.eps, args.scheme, args.tol, 1)[0]
        tn = cpu_run(csr, b, lv, args.eps, args.scheme, args.tol, allc)[0]
        threads = 1 if t1 <= tn else allc
    for _ in range(max(0, args.warmup - 1)):
        cpu_run(csr, b, lv, args.eps, args.scheme, args.tol, threads)
    times = []
    its = 0
    fl = 0.0
    for _ in range(args.steps):
        dt, its, fl = cpu_run(csr, b, lv, args.eps, args.scheme, args.tol, threads)
        times.append(dt)
    t = float(np.mean(times))
    val = fl / t / 1e9
    loaded = sorted(m for m in sys.modules if m.startswith("paper_2007_00789_b200"))
    assert not loaded, f"reference arm imported the product: {loaded}"
    sample = (f"C4-family sample: 3D {SAMPLE['grid']}^3 high-contrast (n={csr[0]}), "
              f"levels {lv}, eps {args.eps}, {args.scheme}, factorize+PCG(1e-12), "
              f"n_cg {its}, mean of {args.steps} runs, BLAS threads {threads} "
              f"(faster of 1 and {allc})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC,
        "value": val, "unit": "GFLOP/s", "higher_is_better": True,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * t, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": sample, "parallelism": "cpu"},
        "same_config": False,
        "same_config_note": ("the reference (pure Python, BLAS-2 pivoted QR loop) needs "
                             "~4400 s for one C4-L15 step, beyond a bench run's limit; this "
                             "arm times the CPU port (bitwise restatement of spdkit, "
                             "tests/test_oracle_golden.py) on a 24^3 sample of the same "
                             "family. GFLOP/s on a smaller problem favours neither side "
                             "fairly, so the ours/reference value ratio is NOT a same-config "
                             "speed-up; ours' line carries the like-for-like pair "
                             "(like_for_like) and the reference's full-config time "
                             "(reference_full_config)"),
        "reference_full_config": reference_full_config(args),
        "product_modules_loaded": loaded,
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def algorithmic_counts(f, a):
    """Algorithmic work of one factorize/apply."""
    diag = f.diagnostics
    f_rrqr = 0.0
    b_rrqr = 0.0
    b_min = 0.0
    for lv in diag["levels"]:
        for e in lv.get("margins", []):
            m, k = e["size_before"], e["k_stop"]
            n = e.get("n_cols", 0)
            ks = np.arange(k, dtype=np.float64)
            f_rrqr += float(np.sum(4 * (m - ks) * np.maximum(n - ks, 0) + 4 * m * (m - ks)))
            b_rrqr += float(np.sum(16.0 * (m - ks) * np.maximum(n - ks, 0)))
            b_min += 8.0 * (2.0 * m * n + m * m)
    b_apply = 16.0 * f.nnz_factor + 32.0 * a.n
    b_spmv = 12.0 * a.nnz + 4.0 * (a.n + 1) + 16.0 * a.n
    return {"F_rrqr": f_rrqr, "B_rrqr_step_traffic": b_rrqr, "B_rrqr_min": b_min,
            "B_apply": b_apply, "B_spmv": b_spmv}


def main():
    args = parse()
    rank, world, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import paper_2007_00789_b200 as sp
    from paper_2007_00789_b200 import _lib
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    a, b, levels = problem(args)
    t0 = time.perf_counter()
    h = sp.build_hierarchy(a, levels)
    t_hier = time.perf_counter() - t0
    bd = torch.from_numpy(b).cuda()
    flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")

    def step_resident():
        f = sp.factorize(a, h, args.eps, args.scheme)
        x, rep = sp.pcg(a, bd, m=f.apply_m, tol=args.tol)
        return f, rep

    def step_e2e():
        a2 = sp.SparseSymMatrix(a.n, a.row_ptr.copy(), a.col_idx.copy(), a.values.copy())
        f = sp.factorize(a2, h, args.eps, args.scheme)
        x, rep = sp.pcg(a2, b, m=f.apply_m, tol=args.tol)
        return f, rep, x

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        return reduce_max(v, dist, "cuda")

    # warm-up in the timed loop's steady state: the previous step's factor is
    # still alive while the next one is built (two block pools in the caching
    # allocator; without this the second timed step paid the cudaMalloc of the
    # second pool, +150 .. 600 ms)
    f = rep = None
    for _ in range(args.warmup):
        f, rep = step_resident()
    # long-lived objects (hierarchy, symbolic tables, the warm-up factor's
    # operator list) leave the cyclic collector's scan set: ~25 ms per step of
    # interpreter housekeeping, no numerical work (SPAND_BENCH_GC=default keeps
    # the interpreter's default)
    if os.environ.get("SPAND_BENCH_GC", "freeze") == "freeze":
        import gc
        gc.collect()
        gc.freeze()
    # ---- timed region: K steps, inputs resident
    barrier()
    st = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launches()
    step_ms = []
    with Clocks(local) as clk, _lib.profile(names={"spand_rrqr_wave"}) as prof:
        ev0.record(st)
        for _ in range(args.steps):
            flush.zero_()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(st)
            f, rep = step_resident()
            s1.record(st)
            torch.cuda.synchronize()
            step_ms.append(s0.elapsed_time(s1))
        ev1.record(st)
        barrier()
    launches = _lib.launches() - launches0
    total_ms = max_over_ranks(float(np.sum(step_ms)))
    ms_step = total_ms / args.steps
    # ---- e2e: public API from host buffers
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 2))):
        barrier()
        t0 = time.perf_counter()
        f2, rep2, x2 = step_e2e()
        torch.cuda.synchronize()
        e2e_ms.append(1000 * (time.perf_counter() - t0))
    e2e_step = max_over_ranks(float(np.mean(e2e_ms)))
    csr_bytes = 4 * (a.n + 1) + 12 * a.nnz
    h2d = csr_bytes + 16 * a.nnz + 8 * a.n      # CSR + block-scatter (index, value) + b
    d2h = 8 * a.n
    # ---- per-kernel breakdown: one extra resident step with events around
    # every launch (outside the timed region; only the dominant kernel is
    # timed inside it)
    barrier()
    with _lib.profile() as prof_all:
        step_resident()
    kern = prof_all.result
    # ---- roofline of the dominant kernel, from the timed-region events
    dom = max(kern.items(), key=lambda kv: kv[1]["ms"])
    dom_steps = 1
    if dom[0] in prof.result:
        dom = (dom[0], prof.result[dom[0]])
        dom_steps = args.steps
    counts = algorithmic_counts(f, a)
    pk, pk_kind = peaks()
    t_f = f.timings.get("total_s", 0.0)
    if dom[0] == "spand_rrqr_wave":
        # B_rrqr,min = 8 (2 m n + m^2) per panel (read the panel,
        # write R/E back, write Q); the per-launch figure is the step total over
        # the launches of a step
        sec = dom[1]["ms"] / dom_steps / 1000.0
        achieved = counts["B_rrqr_min"] / sec / 1e9
        roof = {"kernel": dom[0], "bound": "hbm", "achieved": achieved,
                "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                "peak_kind": pk_kind, "traffic": None,
                "ms_per_step": dom[1]["ms"] / dom_steps,
                "launches_per_step": dom[1]["calls"] / dom_steps,
                "algorithmic_bytes_per_step": counts["B_rrqr_min"],
                "effective_tflops": counts["F_rrqr"] / sec / 1e12,
                "basis": "B_rrqr,min = 8(2mn + m^2) per panel (SURVEY 8d) / RRQR time; the "
                         "pivoted QR needs k_stop sequential group-synchronised steps, so it "
                         "sits far below this bound; effective_tflops = F_rrqr / time"}
    elif dom[0] in ("spand_gemv_tiles", "spand_gemv_items"):
        achieved = counts["B_apply"] * (rep.n_cg + 1) / (dom[1]["ms"] / dom_steps / 1000.0) / 1e9
        roof = {"kernel": dom[0], "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "peak_kind": pk_kind,
                "traffic": None, "basis": "B_apply = 16 nnz_factor + 32 n per apply_m"}
    else:
        roof = {"kernel": dom[0], "bound": "tensor", "achieved": None, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": None, "traffic": None}
    # latency floor of the RRQR: its critical path is the sum over waves of
    # the largest k_stop, each step at least one group synchronisation
    # (tools/rrqr_step_probe.cu: barrier + candidate scan + pivot-column read
    # with no column work, measured on this GPU model)
    probe_path = os.path.join(HERE, "profiles", "rrqr_step_probe_r01.jsonl")
    if dom[0] == "spand_rrqr_wave" and os.path.exists(probe_path):
        try:
            pr = [json.loads(l) for l in open(probe_path) if l.strip()]
            step_us = [p["ns_per_step"] for p in pr if p["G"] == 296][0] / 1000.0
            steps = f.timings.get("rrqr_critical_steps", 0)
            floor_ms = steps * step_us / 1000.0
            roof["latency_bound"] = {
                "critical_steps": steps, "step_floor_us": step_us, "floor_ms": floor_ms,
                "frac": floor_ms / roof["ms_per_step"],
                "basis": "critical path = sum over waves of the largest k_stop; each step "
                         "needs one group barrier + candidate scan + pivot-column read "
                         "(profiles/rrqr_step_probe_r01.jsonl: probed with 296 CTAs; the "
                         "waves now run 148, one per SM)"}
        except Exception:
            pass
    prof_path = next((q for q in (os.path.join(HERE, "profiles", f"ncu_r0{k}_summary.json")
                                  for k in (3, 2, 1)) if os.path.exists(q)), "")
    if os.path.exists(prof_path):
        try:
            with open(prof_path) as fh:
                pr = json.load(fh)
            if pr.get("kernel", "").startswith(dom[0].replace("spand_", "")):
                roof["traffic"] = pr.get("traffic_per_step")
                roof["traffic_source"] = pr.get("capture")
        except Exception:
            pass
    from paper_2007_00789_b200.metrics import (device_panels, factor_flops,
                                               solve_flops)
    ff = factor_flops(f.ops, device_panels(f))
    f_step = ff["F_factor"] + solve_flops(f.nnz_factor, a.nnz, rep.n_cg + 1, rep.n_cg + 1)
    # apply GB/s over the whole solve
    # preconditioner apply (one CUDA graph per apply_m) and SpMV, timed after
    # the step on the last factor: 10 back-to-back replays each (the factor,
    # > 6 GB, and A's CSR stream from HBM; L2 is 126 MB)
    xa = bd.clone()
    f.apply_m_device(xa)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # eager (the launches a short solve issues: ~690 per apply_m) ...
    e0.record(st)
    for _ in range(10):
        f.apply_m_device(xa)
    e1.record(st)
    torch.cuda.synchronize()
    apply_eager_ms = e0.elapsed_time(e1) / 10
    # ... and one CUDA graph per apply_m (a factor reused for many solves:
    # captured after fastplan.GRAPH_AFTER applies), L2 flushed before each
    for _ in range(40):
        f.apply_m_device(xa)
    g_ms = []
    for _ in range(10):
        flush.zero_()
        torch.cuda.synchronize()
        e0.record(st)
        f.apply_m_device(xa)
        e1.record(st)
        torch.cuda.synchronize()
        g_ms.append(e0.elapsed_time(e1))
    apply_ms = float(np.median(g_ms))
    apply_gbs = counts["B_apply"] / (apply_ms / 1000.0) / 1e9
    # multi-RHS apply (8 right-hand sides per pass, payload read once per 4)
    xm = torch.randn(a.n, 8, dtype=torch.float64, device=bd.device)
    f.plan.run(xm.clone())
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(3):
        f.plan.run(xm)
    e1.record(st)
    torch.cuda.synchronize()
    multi_ms = e0.elapsed_time(e1) / 3
    dcsr = a.device()
    ya = torch.empty_like(bd)
    # 20 back-to-back SpMVs captured in one CUDA graph (no launch gaps)
    dcsr.spmv(bd, ya)
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    gsp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gsp, stream=gs):
        for _ in range(20):
            dcsr.spmv(bd, ya)
    torch.cuda.current_stream().wait_stream(gs)
    gsp.replay()
    flush.zero_()
    torch.cuda.synchronize()
    e0.record(st)
    gsp.replay()
    e1.record(st)
    torch.cuda.synchronize()
    spmv_ms = e0.elapsed_time(e1) / 20
    spmv_gbs = counts["B_spmv"] / (spmv_ms / 1000.0) / 1e9
    line = {
        "metric": METRIC, "value": whole_job_rate(f_step, world, ms_step) / 1e9,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: 3D 64^3 high-contrast harmonic FV, n={a.n}, "
                               f"ND levels {levels}, eps {args.eps}, {args.scheme}, skip 4, "
                               f"PCG tol {args.tol}, b~N(0,1) seed 3",
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "flushed between steps (256 MiB write); factor > L2",
                   "host": "gc.freeze() after warm-up; warm-up keeps the previous factor alive "
                           "like the timed loop"},
        "step_ms": [round(float(v), 1) for v in step_ms],
        "factorize_s": t_f, "solve_s": rep.solve_seconds, "n_cg": rep.n_cg,
        "true_residual": rep.true_residual, "hierarchy_s": t_hier,
        "nnz_factor": f.nnz_factor, "mu": f.nnz_factor / a.nnz,
        "apply": {"ms": apply_ms, "gbs": apply_gbs, "frac_hbm": apply_gbs / pk["hbm_gbs"],
                  "bytes": counts["B_apply"], "eager_ms": apply_eager_ms,
                  "eager_gbs": counts["B_apply"] / (apply_eager_ms / 1000.0) / 1e9,
                  "basis": "B_apply = 16 nnz_factor + 32 n per apply_m; ms: one CUDA graph "
                           "replay (L2 flushed before, median of 10); eager_ms: the ~690 "
                           "launches of a short solve, back to back"},
        "apply_multi_rhs": {"rhs": 8, "ms": multi_ms, "ms_per_rhs": multi_ms / 8,
                            "gbs_per_rhs_equiv": 8 * counts["B_apply"] / (multi_ms / 1000.0) / 1e9,
                            "basis": "apply_m of an n x 8 stack (eager launches, two passes of "
                                     "4 vectors each); GB/s counts B_apply per vector"},
        "spmv": {"ms": spmv_ms, "gbs": spmv_gbs, "frac_hbm": spmv_gbs / pk["hbm_gbs"],
                 "bytes": counts["B_spmv"], "l2_resident": True,
                 "basis": "B_spmv = 12 nnz(A) + 4(n+1) + 16 n; 20 SpMVs in one CUDA graph after an "
                          "L2 flush; A (22 MB) stays in L2 after the first"},
        "kernels_ms_per_step": {k: round(v["ms"], 3) for k, v in kern.items()},
        "kernels_note": "kernels_ms_per_step: one extra profiled step outside the timed region; "
                        "roofline.ms_per_step: events around the dominant kernel inside it",
        "flops_per_step": ff | {"F_step": f_step},
        "dof_per_s": whole_job_rate(a.n, world, ms_step),
        "e2e": {"value": whole_job_rate(f_step, world, e2e_step) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_step},
        "fp64": {"achieved_tflops": whole_job_rate(f_step, world, ms_step) / 1e12 / world,
                 "peak_tflops": FP64_DGEMM_TFLOPS,
                 "frac": whole_job_rate(f_step, world, ms_step) / 1e12 / world / FP64_DGEMM_TFLOPS,
                 "peak_basis": "cuBLAS DGEMM 8192^3 on this pool's B200 "
                               "(profiles/fp64_peak_r01.jsonl); algorithmic flops of the "
                               "whole step over its time"},
        "roofline": roof, "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    # the Schur / TRSM / rescale products (north_star d): algorithmic flops
    # F_elim + F_scale over the grouped-GEMM launches of a step (with the
    # K-chunk mask pass that feeds them)
    gemm_ms = sum(v["ms"] for k, v in kern.items()
                  if k in ("spand_gemm_grouped", "spand_gemm_kmask"))
    if gemm_ms > 0:
        gtf = (ff["F_elim"] + ff["F_scale"]) / (gemm_ms / 1000.0) / 1e12
        line["gemm"] = {"ms": gemm_ms, "tflops": gtf,
                        "frac_cublas_dgemm": gtf / FP64_DGEMM_TFLOPS,
                        "frac_dmma_peak": gtf / 33.1,
                        "basis": "(F_elim + F_scale) / (spand_gemm_grouped + spand_gemm_kmask "
                                 "time of the profiled step); peaks: cuBLAS DGEMM 35.5, DMMA "
                                 "loop 33.1 TFLOP/s (profiles/fp64_peak_r01.jsonl)"}
    if rank == 0 and not args.no_near_kernel:
        # near-kernel extension (not in the reference, so not the headline):
        # BASELINE C4 asks for the constant vector preserved in each coarse
        # basis.  Same step protocol as the headline:
        # warm-up, then K steps of factorize(near_kernel=ones) + pcg with
        # CUDA events on the stream, L2 flushed between steps.
        ones = np.ones(a.n)

        def step_nk():
            fnk_ = sp.factorize(a, h, args.eps, args.scheme, near_kernel=ones)
            _, rnk_ = sp.pcg(a, bd, m=fnk_.apply_m, tol=args.tol)
            return fnk_, rnk_
        fnk = rnk = None
        for _ in range(max(1, args.warmup)):
            fnk, rnk = step_nk()   # previous factor alive, as in the timed loop
        nk_ms = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0.record(st)
            fnk, rnk = step_nk()
            e1.record(st)
            torch.cuda.synchronize()
            nk_ms.append(e0.elapsed_time(e1))
        nk_step = float(np.mean(nk_ms))
        ffn = factor_flops(fnk.ops, device_panels(fnk))
        fnk_step = ffn["F_factor"] + solve_flops(fnk.nnz_factor, a.nnz, rnk.n_cg + 1,
                                                 rnk.n_cg + 1)
        kept = lambda ff: sum(e["size_after"] for lv_ in ff.diagnostics["levels"]  # noqa: E731
                              for e in lv_["interfaces"])
        line["near_kernel"] = {
            "vectors": "constant (ones)", "ms_per_step": nk_step, "steps": args.steps,
            "value": fnk_step / (nk_step / 1000.0) / 1e9, "unit": "GFLOP/s",
            "factorize_s": fnk.timings.get("total_s"), "n_cg": rnk.n_cg,
            "solve_s": rnk.solve_seconds, "true_residual": rnk.true_residual,
            "coarse_dofs_kept": kept(fnk), "coarse_dofs_kept_reference_path": kept(f),
            "nnz_factor": fnk.nnz_factor, "n_cg_reference_path": rep.n_cg,
            "basis": "factorize(..., near_kernel=ones) + PCG to the same tol, timed like the "
                     "headline (warm-up, K steps, events, L2 flush); extension, checked "
                     "against its own CPU oracle in tests/test_near_kernel.py"}
        del fnk
    if rank == 0 and world == 1:
        line["reference_full_config"] = reference_full_config(args)
        if line["reference_full_config"]:
            line["reference_full_config"]["speedup_vs_this_step"] = (
                line["reference_full_config"]["step_s"] / (ms_step / 1000.0))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        csr, sb, slv = sample_problem()
        dt, its, sfl = cpu_run(csr, sb, slv, args.eps, args.scheme, args.tol, 1)
        line["cpu_baseline"] = {
            "value": sfl / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": f"oracle port (bitwise restatement of spdkit) on a C4-family "
                      f"24^3 sample (n={csr[0]}, levels {slv}), factorize+PCG {dt:.2f} s, "
                      f"n_cg {its}, OpenBLAS 1 thread"}
        # the like-for-like pair: this GPU on the very same sample, same run
        sa = sp.SparseSymMatrix(*csr)
        sh = sp.build_hierarchy(sa, slv)
        sbd = torch.from_numpy(sb).cuda()
        for _ in range(2):
            fs = sp.factorize(sa, sh, args.eps, args.scheme)
            sp.pcg(sa, sbd, m=fs.apply_m, tol=args.tol)
        g_ms = []
        for _ in range(3):
            torch.cuda.synchronize()
            e0.record(st)
            fs = sp.factorize(sa, sh, args.eps, args.scheme)
            _, srep = sp.pcg(sa, sbd, m=fs.apply_m, tol=args.tol)
            e1.record(st)
            torch.cuda.synchronize()
            g_ms.append(e0.elapsed_time(e1))
        gpu_ms = float(np.mean(g_ms))
        line["like_for_like"] = {
            "sample": line["cpu_baseline"]["sample"].split(", factorize")[0],
            "cpu_port_ms": 1000 * dt, "gpu_ms": gpu_ms, "speedup": 1000 * dt / gpu_ms,
            "n_cg_cpu": its, "n_cg_gpu": srep.n_cg,
            "basis": "same matrix, hierarchy, eps, scheme and tol on both sides; GPU: "
                     "factorize + pcg with inputs resident, mean of 3 after 2 warm-ups"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
