#!/usr/bin/env python
"""bench.py -- screened box-constrained least squares on B200.

Headline workload (BASELINE.json config 3, the largest fp64 configuration that
fits one GPU and the one the metric's "achieved HBM GB/s" is meaningful for):
NNLS, A 10000 x 50000 fp64 (4 GB, Uniform[0,1) entries, unit columns), x0 2%
nonzeros |N(0,1)|, 30 dB SNR, accelerated projected gradient (FISTA +
function-value restart) with gap-safe screening every 10 iterations, solved to
a certified duality gap <= 1e-6.  One bench "step" = one full solve from
x = clip(0, l, u) (setup, power iteration, all rounds, the certified gap).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3]
    python bench.py --impl reference ...      # the CPU reference arm

JSON line keys: value = screened FISTA iterations per second over whole solves
(inputs resident in HBM), ms_per_step = time-to-gap, e2e = the same through the
public API from pinned host buffers (H2D of A, y, bounds and D2H of x, theta
inside the timed region), roofline = the fused FISTA pass kernel timed live
with CUDA events, cpu_baseline = the unmodified reference (baseline/_ref) on
the host cores when it is installed, else the oracle port.  Extra keys
measure what screening buys on the GPU (time_to_gap_unscreened_s, the
reference's off/on protocol, bench.py:96-115) and, for config 3, the FISTA
restart rule BASELINE states (time_to_gap_stated_restart_s: restart on an
objective increase only).
"""

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

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
def traj_path(cfg_id):
    """Preserved-count trajectory of the GPU solve of a config (the CPU arm's
    iteration weights), written with --write-trajectory."""
    return os.path.join(ROOT, "profiles", f"cfg{cfg_id}_trajectory.json")
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--rounds", type=int, default=8, help="config 5: rounds (x10 FISTA steps) per step")
    ap.add_argument("--check-every", type=int, default=0,
                    help="config 5: rounds between convergence checks / host round trips (0: min(rounds, 16))")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=4, help="solves in the e2e leg (after one untimed)")
    ap.add_argument("--no-study", action="store_true", help="skip the screening-off / stated-restart solves")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--write-trajectory", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="configs 3/4: take the NCCL column-sharded path even at N=1 (exercises the N>1 code)")
    ap.add_argument("--cfg4-rounds", type=int, default=100,
                    help="config 4: rounds (x10 PG passes + screening) per step; BASELINE gives it no gap target")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        with open(PEAKS_PATH) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", pk
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        # sampling period (BX_SMI_MS overrides; A/B on config 2 showed no
        # measurable interference at 200 ms)
        self.period_ms = int(os.environ.get("BX_SMI_MS", "200"))
        self.proc = None
        self.lines = []
        self.t = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, util_floor=0.0):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# the CPU side: oracle port timed on the host cores (cpu_baseline / reference arm)
# ---------------------------------------------------------------------------
# ---------------------------------------------------------------------------
# the unmodified reference (baseline/_ref, installed from /root/reference/pkg)
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_module():
    """The reference package ``boxscreen`` from baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "boxscreen")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import boxscreen
        import boxscreen.solvers  # noqa: F401
        return boxscreen
    except Exception:
        return None


def ref_step_rate(bs, inst, k_bins, budget_s, kmax=None):
    """The reference's own per-iteration work on the solve's trajectory:
    ``pg_step`` (solvers.py:101-116: clip, A_act x, A_act' r -- the two GEMVs
    an iteration costs in the reference; it has no FISTA, whose oracle step is
    the same two products) timed on the reference's Workspace
    (solvers.py:48-65) over k-column preserved sets at the solve's
    preserved-count bins, weighted by the iterations the solve spends there.
    Bins wider than ``kmax`` columns are timed on kmax and scaled by k / kmax
    (GEMVs are linear in k).  Returns (iterations/s, details)."""
    a, y, lo, hi = inst.a, inst.y, inst.lower, inst.upper
    n = a.shape[1]
    perm = np.random.default_rng(1).permutation(n)
    total_it = sum(it for _, it in k_bins)
    per_bin = budget_s / max(1, len(k_bins))
    details, tsum = [], 0.0
    for k, it in k_bins:
        kt = min(k, kmax or k)
        keep = np.sort(perm[:kt])
        p = bs.Problem(np.asarray(a[:, keep], dtype=np.float64), y, lo[keep], hi[keep])
        st = bs.ScreeningState(p)
        ws = bs.solvers.Workspace(p, st, bs.PrimalPoint(np.clip(np.zeros(kt), lo[keep], hi[keep])))
        eta = 1e-6  # timing only (a small step keeps the objective monotone); cost is step-independent
        bs.solvers.pg_step(ws, eta, 1)  # warm
        t0 = time.perf_counter()
        done = 0
        while True:
            bs.solvers.pg_step(ws, eta, 1)
            done += 1
            el = time.perf_counter() - t0
            if el > per_bin or done >= it:
                break
        sec = el / done * (k / kt)
        details.append(dict(k=int(k), timed_columns=int(kt), iterations_in_solve=int(it), timed_iterations=done,
                            sec_per_iteration=sec))
        tsum += it * sec
        del ws, st, p
    return total_it / tsum, details


def ref_solve_rate(bs, inst, screening, max_rounds=None):
    """The reference's ``solve`` (driver.py:131-256) on the config, timed by
    its own convention (trace[-1].elapsed, the offline-gap rule with screening
    off; bench.py:86-93).  Returns (iterations/s, elapsed, result)."""
    p = bs.Problem(inst.a, inst.y, inst.lower, inst.upper)
    cfg = bs.SolverConfig(kind=inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol,
                          max_rounds=max_rounds or 10 ** 6)
    res = bs.solve(p, cfg, screening=screening)
    el = res.trace[-1].elapsed
    iters = res.rounds * inst.inner_passes
    return iters / el, el, res


def cpu_rate(inst, k_bins, budget_s, passes=None, kmax=8000):
    """Oracle FISTA iterations/s over the solve's preserved-set trajectory.

    ``k_bins`` = [(k, iterations)] -- how many iterations the screened solve
    spends at each preserved count.  For each bin the oracle's FISTA passes
    (oracle/boxscreen_oracle.py:apg_passes, the reference's two-GEMV
    Workspace arithmetic) are timed on a k-column working set; the rate is
    total iterations / sum(iterations_b * seconds_per_iteration(k_b)).
    Bins wider than ``kmax`` columns are timed on ``kmax`` of them and scaled
    by k / kmax (the passes are GEMVs, linear in k), so the fp64 working set
    stays bounded (config 4's shard is 10 GB in fp64).  The oracle always runs
    in fp64 (the reference's arithmetic).  Returns (rate, details).
    """
    from oracle.boxscreen_oracle import ActiveView, apg_passes, cd_passes, pg_passes
    a, y, lo, hi = inst.a, inst.y, inst.lower, inst.upper
    passes = passes or inst.inner_passes
    if inst.kind == "pg":
        step_fn = lambda w, eta, p, mom: pg_passes(w, eta, p)  # noqa: E731
    elif inst.kind == "cd":
        step_fn = lambda w, eta, p, mom: cd_passes(w, p)  # noqa: E731
    else:
        step_fn = apg_passes
    n = a.shape[1]
    norms = np.ones(n)
    perm = np.random.default_rng(1).permutation(n)
    total_it = sum(it for _, it in k_bins)
    per_bin = budget_s / max(1, len(k_bins))
    details = []
    tsum = 0.0
    x_full = np.zeros(n)
    for k, it in k_bins:
        kt = min(k, kmax)
        keep = np.sort(perm[:kt])
        sub = np.asarray(a[:, keep], dtype=np.float64, order="F")
        w = ActiveView(sub, y, lo[keep], hi[keep], norms[keep], np.zeros(a.shape[0]), x_full[keep], np.arange(kt))
        eta = 0.5 / (0.75 * kt + 10.0)  # timing only: cost does not depend on the step
        mom = [1.0]
        t0 = time.perf_counter()
        done = 0
        while True:
            step_fn(w, eta, passes, mom)
            done += passes
            el = time.perf_counter() - t0
            if el > per_bin or done >= it:
                break
        sec_per_it = el / done * (k / kt)
        details.append(dict(k=int(k), timed_columns=int(kt), iterations_in_solve=int(it), timed_iterations=done,
                            sec_per_iteration=sec_per_it))
        tsum += it * sec_per_it
        del w
    return total_it / tsum, details


def k_bins_from_trace(trace_arrays, passes, nbins=6):
    """Bin the solve's iterations by preserved count (count in force during the round)."""
    ks = [int(r["preserved_count"]) for r in trace_arrays]
    start = [ks[0]] + ks[:-1]  # preserved count during round i (before its own screening)
    n0 = max(start)
    counts = {}
    for k in start:
        counts[k] = counts.get(k, 0) + passes
    items = sorted(counts.items())
    # quantile bins weighted by iterations
    total = sum(c for _, c in items)
    bins, acc, cur_k_w, cur_it = [], 0, 0.0, 0
    edge = total / nbins
    for k, c in items:
        cur_k_w += k * c
        cur_it += c
        acc += c
        if acc >= edge * (len(bins) + 1) or (k, c) == items[-1]:
            bins.append((max(1, int(round(cur_k_w / cur_it))), cur_it))
            cur_k_w, cur_it = 0.0, 0
    del n0
    return bins


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return os.cpu_count(), model


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        for inf in threadpool_info():
            if inf.get("internal_api") in ("openblas", "mkl", "blis"):
                return int(inf.get("num_threads", 0))
    except Exception:
        pass
    return os.cpu_count()


# ---------------------------------------------------------------------------
CFG4_COLS_PER_GPU = 62500  # BASELINE config 4: 500,000 columns over 8 GPUs (weak scaling unit)
# BASELINE config 4 states no gap target (its check is the 1e-4 objective
# agreement with fp64) and plain PG needs millions of steps to a 1e-6 gap on
# this coherent matrix, so a step is a fixed budget of screened rounds
CFG4_STEP = "fixed budget: --cfg4-rounds rounds of 10 PG passes + the screening pass (no gap target in config 4)"


def make_instance(cfg_id):
    """The single-GPU workload of a config.  Config 4 is the weak-scaling
    unit: 20000 x 62,500 fp32 (its columns of the 8-GPU 500,000-column run)."""
    from paper_2202_07258_b200.generate import CONFIGS, Instance, make_config, sparse_nnls_block
    if cfg_id != 4:
        return make_config(cfg_id)
    c = CONFIGS[4]
    n = CFG4_COLS_PER_GPU
    a, y, lo, hi, x0 = sparse_nnls_block(c["m"], n, c["density"], c["snr"], 0, n, lambda v: v, dtype=np.float32)
    return Instance(c["name"], a, y, lo, hi, x0, c["kind"], c["inner_passes"], c["gap_tol"])


def config_block(cfg_id, inst):
    from paper_2202_07258_b200.generate import CONFIGS
    c = CONFIGS[cfg_id]
    extra = {"n_per_gpu": CFG4_COLS_PER_GPU, "parallelism": "1 GPU = one 62,500-column shard of the 8-GPU run"} \
        if cfg_id == 4 else {}
    return {"workload": c["name"], **extra, "m": int(inst.a.shape[0]), "n": int(inst.a.shape[1]), "solver": inst.kind,
            "inner_passes": inst.inner_passes, "gap_tol": inst.gap_tol, "screening": True,
            "problem": "NNLS" if np.isinf(inst.upper).all() else "BVLS", "seed": 0,
            "l2_policy": "inputs larger than L2 (A = %.1f GB > 126 MB L2)" % (inst.a.nbytes / 1e9)
            if inst.a.nbytes > 126e6 else "working set L2-resident (reported, not flushed)",
            "step": CFG4_STEP if cfg_id == 4 else "one full solve to certified gap <= gap_tol"}


STEP_LABEL = {"pg": "PG passes", "apg": "FISTA passes", "cd": "CD sweeps", "active-set": "active-set iterations"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    bs = reference_module()
    if bs is not None:
        return run_reference_unmodified(args, bs, world)
    inst = make_instance(args.config)
    try:
        with open(traj_path(args.config)) as fh:
            traj = json.load(fh)
        if traj.get("config") != args.config:
            raise ValueError("trajectory of another config")
        bins = [tuple(b) for b in traj["k_bins"]]
        src = f"preserved-count trajectory of the GPU solve (profiles/cfg{args.config}_trajectory.json)"
    except Exception:
        bins = [(inst.a.shape[1], 100)]
        src = "unscreened working set (no trajectory file)"
    per_step_budget = max(5.0, args.cpu_budget / max(1, args.steps))
    for _ in range(args.warmup):
        pass  # CPU arm: warm-up is the first (untimed) view construction inside cpu_rate
    rates, details = [], None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, details = cpu_rate(inst, bins, per_step_budget)
        rates.append(r)
    wall = time.perf_counter() - t0
    rate = float(np.median(rates))
    cores, model = cpu_info()
    thr = blas_threads()
    sample = (f"oracle {STEP_LABEL[inst.kind]} (numpy/OpenBLAS, reference Workspace arithmetic) timed at "
              f"{len(bins)} preserved-count bins weighted by {src}; "
              f"{sum(d['timed_iterations'] for d in details)} iterations per step")
    line = {"impl": "reference", "metric": metric_name(args.config), "value": rate, "unit": unit_name(args.config),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * wall / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong" if args.config in (3, 5) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config recipe)",
            "config": config_block(args.config, inst),
            "cpu_baseline": {"value": rate, "unit": unit_name(args.config), "cores": thr, "kind": "port", "sample": sample,
                             "cpu_model": model, "nproc": cores, "bins": details},
            "e2e": {"value": rate, "unit": unit_name(args.config), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def load_bins(cfg_id, inst):
    try:
        with open(traj_path(cfg_id)) as fh:
            traj = json.load(fh)
        if traj.get("config") != cfg_id:
            raise ValueError("trajectory of another config")
        return ([tuple(b) for b in traj["k_bins"]],
                f"preserved-count trajectory of the GPU solve (profiles/cfg{cfg_id}_trajectory.json)")
    except Exception:
        return [(inst.a.shape[1], 100)], "unscreened working set (no trajectory file)"


def run_reference_unmodified(args, bs, world):
    """--impl reference with the unmodified reference installed in
    baseline/_ref: its own code on the host cores (all BLAS threads).
    Configs 3 / 4 (no FISTA / no fp32 in the reference): its pg_step on the
    solve's preserved-count trajectory; configs 1 / 2: its solve() on a
    bounded number of rounds per step."""
    inst = make_instance(args.config)
    cores, model = cpu_info()
    thr = blas_threads()
    extra = {}
    t0 = time.perf_counter()
    rates = []
    if args.config in (3, 4):
        bins, src = load_bins(args.config, inst)
        budget = max(3.0, args.cpu_budget / max(1, args.steps))
        kmax = 16000 if args.config == 4 else None
        for _ in range(args.steps):
            r, det = ref_step_rate(bs, inst, bins, budget, kmax=kmax)
            rates.append(r)
        sample = (f"unmodified reference pg_step (solvers.py:101-116, 2 GEMVs per iteration) on its Workspace at "
                  f"{len(bins)} preserved-count bins weighted by {src}; "
                  f"{sum(d['timed_iterations'] for d in det)} iterations per step"
                  + ("; fp64 (the reference copies A to fp64), bins > 16000 columns scaled" if args.config == 4 else ""))
        extra["bins"] = det
    else:
        rounds = 2000 if args.config == 1 else 100
        for _ in range(args.steps):
            r, _, _ = ref_solve_rate(bs, inst, True, max_rounds=rounds)
            rates.append(r)
        sample = (f"unmodified reference solve() (driver.py:131-256), first {rounds} screened rounds per step, "
                  f"timed by trace[-1].elapsed")
    wall = time.perf_counter() - t0
    rate = float(np.median(rates))
    line = {"impl": "reference", "metric": metric_name(args.config), "value": rate, "unit": unit_name(args.config),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * wall / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong" if args.config in (3, 5) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config recipe)",
            "config": config_block(args.config, inst),
            "cpu_baseline": {"value": rate, "unit": unit_name(args.config), "cores": thr, "kind": "reference",
                             "sample": sample, "cpu_model": model, "nproc": cores, **extra},
            "e2e": {"value": rate, "unit": unit_name(args.config), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def unit_name(cfg_id):
    """Config 4's unit is one 62,500-column shard iteration (weak scaling)."""
    return "shard-iters/s" if cfg_id == 4 else "iters/s"


def metric_name(cfg_id):
    return ("screened iters/s & time-to-gap<=1e-6 (m x n fp64); achieved HBM GB/s vs peak "
            f"[config {cfg_id}]")


NCU_TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def ncu_traffic(cfg_id):
    """DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
    dominant kernel from the committed `ncu --set full` capture of this
    config (profiles/ncu_traffic.json, one launch), with that launch's
    algorithmic bytes, so traffic / algorithmic shows any re-reads."""
    try:
        with open(NCU_TRAFFIC_PATH) as fh:
            ent = json.load(fh)[str(cfg_id)]
    except Exception:
        return None, None
    t = float(ent["dram_read_bytes"]) + float(ent["dram_write_bytes"])
    info = {"traffic_source": ent["source"], "traffic_kernel": ent["kernel"],
            "traffic_launch_algorithmic": ent.get("algorithmic"),
            "traffic_over_algorithmic": (t / ent["algorithmic"]) if ent.get("algorithmic") else None}
    if ent.get("launch_list"):
        info["launch_list"] = ent["launch_list"]  # ncu --metrics gpu__time_duration.sum of this command
    return t, info


KERNEL_NAMES = {"cd": "k_cd (software-pipelined block-exact cyclic CD on a thread-block cluster)",
                "small_round": "k_round_small (cooperative SM-resident PG/FISTA round)"}


def kernel_name(key):
    return KERNEL_NAMES.get(key, f"k_pass[{key}]")


def roofline_block(prof, cfg_id=None):
    hbm, peak_src, _ = peaks()
    prof = prof or {}
    tot_ms = sum(v["ms"] for v in prof.values()) or 1.0
    dom_name = max(prof, key=lambda k: prof[k]["ms"]) if prof else None
    dom = prof.get(dom_name, {"ms": 0.0, "bytes": 0.0, "launches": 0})
    achieved = dom["bytes"] / (dom["ms"] / 1e3) / 1e9 if dom["ms"] > 0 else 0.0
    traffic, tinfo = ncu_traffic(cfg_id)
    out = {"bound": "hbm", "kernel": kernel_name(dom_name), "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
            "launches": dom["launches"], "avg_launch_us": 1e3 * dom["ms"] / max(1, dom["launches"]),
            "share_of_kernel_time": dom["ms"] / tot_ms,
            "bytes_per_launch_avg": dom["bytes"] / max(1, dom["launches"]),
            "algorithmic_bytes": "8*m per streamed column + per-column state + row vectors (DESIGN.md)",
            "passes_per_iteration": 1,
            "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                            "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None}
                        for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}}
    if tinfo:
        out.update(tinfo)
    if out["frac"] > 1.0:
        out["frac_note"] = ("the measured peak is a read + write copy (MEASURED_PEAKS.json 'how'); this pass is "
                            "~99.9% reads, which HBM serves faster than a 1:1 read/write mix")
    return out


def run_sharded(args, rank, world, dev):
    """Configs 3 / 4 over `world` GPUs: NCCL column sharding (csrc/bx_core.cu)."""
    import torch
    import torch.distributed as dist
    from paper_2202_07258_b200 import Problem, SolverConfig
    from paper_2202_07258_b200.distributed import column_blocks, solve_distributed
    from paper_2202_07258_b200.generate import CONFIGS, sparse_nnls_block
    c = CONFIGS[args.config]
    m = c["m"]
    n = c["n"] if args.config == 3 else 62500 * world  # config 4: 62,500 columns per GPU (weak)
    c0, c1 = column_blocks(n, world)[rank]

    def reduce_sum(v):
        t = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
        dist.all_reduce(t)
        return t.cpu().numpy()

    dt = np.float32 if args.config == 4 else np.float64
    a_blk, y, lo, hi, _ = sparse_nnls_block(m, n, c["density"], c["snr"], c0, c1, reduce_sum, dtype=dt)
    a_dev = torch.from_numpy(np.ascontiguousarray(a_blk.T)).to(dev)
    tdt = a_dev.dtype
    p = Problem.from_device_storage(a_dev, m, torch.from_numpy(y).to(dev).to(tdt), lo, hi)
    cfg = SolverConfig(kind=c["kind"], inner_passes=c["inner_passes"], gap_tol=c["gap_tol"],
                       max_rounds=args.cfg4_rounds if args.config == 4 else None)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        solve_distributed(p, c0, n, cfg)
    torch.cuda.synchronize()
    results = []
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            results.append(solve_distributed(p, c0, n, cfg))
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    el = torch.tensor([ev0.elapsed_time(ev1) / 1000.0], device=dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    elapsed = float(el.item())
    iters = sum(r.info["iterations"] for r in results)
    launches = sum(r.info["kernel_launches"] for r in results)
    prof_res = solve_distributed(p, c0, n, cfg, profile=True)
    roof = roofline_block(prof_res.info["profile"], args.config)
    e2e = None
    if not args.no_e2e:
        p_host = Problem(a_blk, y, lo, hi, dtype=dt, pin=True)
        h2d = p_host.a_matrix.nbytes + y.nbytes + lo.nbytes + hi.nbytes
        e_it, e_t = 0, 0.0
        for s_ in range(args.steps + 1):
            p_host.release_device()
            dist.barrier()
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            r = solve_distributed(p_host, c0, n, cfg, return_device=False)
            t1.record(stream)
            torch.cuda.synchronize()
            tt = torch.tensor([t0.elapsed_time(t1) / 1000.0], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            if s_ == 0:
                continue
            e_t += float(tt.item())
            e_it += r.info["iterations"]
        e2e = {"value": (world if args.config == 4 else 1) * e_it / e_t,
               "unit": unit_name(args.config), "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(8 * (c1 - c0) + 8 * m), "ms_per_step": 1000.0 * e_t / args.steps,
               "note": "per-rank bytes; every rank uploads its own column block"}
    r0 = results[0]
    # config 4 is weak scaling (62,500 columns per GPU): the whole-job value is
    # shard-iterations/s (world x iterations/s of the global solve), the N=1
    # unit; config 3 is strong scaling of one fixed problem: iterations/s
    agg = world if args.config == 4 else 1
    line = {"metric": metric_name(args.config), "value": agg * iters / elapsed,
            "unit": unit_name(args.config), "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * elapsed / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.config == 3 else "weak", "vs_baseline": None,
            "dtype": "f32" if dt == np.float32 else "f64",
            "data": "synthetic (seeded numpy, BASELINE config recipe; per-rank column blocks of the same draw)",
            "config": {"workload": c["name"], "m": m, "n": n, "solver": c["kind"], "inner_passes": c["inner_passes"],
                       "gap_tol": c["gap_tol"], "screening": True, "parallelism": f"column-sharded x{world}",
                       "exchange": ("per-step reduction: fused reduce + peer-memory exchange kernel (CUDA IPC, "
                                    "NVLink); per-round scalars: NCCL")
                       if os.environ.get("BX_EXCHANGE", "fused") == "fused" else "NCCL allreduces",
                       "l2_policy": "inputs larger than L2",
                       "step": CFG4_STEP if args.config == 4 else "one full solve to certified gap <= gap_tol"},
            "time_to_gap_s": elapsed / args.steps, "converged": all(r.converged for r in results),
            "rounds": r0.rounds, "iterations_per_solve": r0.info["iterations"],
            "final_preserved": r0.trace[-1].preserved_count, "certified_gap": r0.gap, "gpu_launches": launches,
            "roofline": roof, "cpu_baseline": None, "e2e": e2e, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    from paper_2202_07258_b200.distributed import release_comms
    release_comms()
    dist.destroy_process_group()
    return 0


def dgemm_peak(dev, n=8192, reps=5):
    """cuBLAS DGEMM (fp64 tensor cores) measured on this GPU: the roofline
    denominator for the batched DMMA kernel (MEASURED_PEAKS.json has no fp64)."""
    import torch
    a = torch.randn((n, n), dtype=torch.float64, device=dev)
    b = torch.randn((n, n), dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    del a, b
    return best


def config5_instance(k_rhs, k0=0, k1=None):
    from paper_2202_07258_b200.generate import CONFIGS, batched_rhs, bump_dictionary
    c = CONFIGS[5]
    a = bump_dictionary(c["m"], c["n"])
    Y, _ = batched_rhs(a, k_rhs, snr_db=c["snr"])
    k1 = k_rhs if k1 is None else k1
    return a, np.asfortranarray(Y[:, k0:k1])


def run_batched(args, rank, world, dev):
    """Config 5: K = 100,000 right-hand sides over a 200 x 5000 bump dictionary,
    batched FISTA with per-problem screening on fp64 tensor cores; problems
    sharded across ranks with no communication (strong scaling)."""
    import torch
    from paper_2202_07258_b200.batched import solve_batched
    from paper_2202_07258_b200.generate import CONFIGS
    from paper_2202_07258_b200.solvers import auto_step_size
    c = CONFIGS[5]
    K = c["k_rhs"]
    k0, k1 = K * rank // world, K * (rank + 1) // world
    a, Y = config5_instance(K, k0, k1)
    m, n = a.shape
    kl = k1 - k0
    eta = auto_step_size(a, 1.0)
    a_dev = torch.from_numpy(a).to(dev)
    y_dev = torch.from_numpy(np.ascontiguousarray(Y)).to(dev)
    stream = torch.cuda.current_stream(dev)
    rounds = args.rounds
    every = args.check_every if args.check_every > 0 else min(rounds, 16)
    for _ in range(args.warmup):
        solve_batched(a_dev, y_dev, passes=10, rounds=rounds, gap_tol=c["gap_tol"], eta=eta, return_device=True,
                      check_every=every)
    torch.cuda.synchronize()
    res = []
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            res.append(solve_batched(a_dev, y_dev, passes=10, rounds=rounds, gap_tol=c["gap_tol"], eta=eta,
                                     return_device=True, check_every=every))
        e1.record(stream)
        torch.cuda.synchronize()
    el = e0.elapsed_time(e1) / 1000.0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([el], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    its = sum(r.iterations for r in res)
    launches = sum(r.kernel_launches for r in res)
    # algorithmic flops of the work that ran: two products (2 m n K each) per
    # FISTA step, the dual sweep's A'R per round, and the per-coordinate sphere
    # sweep's A'R for the tiles (64 right-hand sides) the per-problem bound
    # did not clear
    flops = sum(r.rounds * (10 * 4.0 + 2.0) * m * n * kl + r.sphere_sweeps * 64 * 2.0 * m * n for r in res) * world
    kern_s = sum(r.round_kernel_ms for r in res) / 1e3
    peak = dgemm_peak(dev)
    achieved = flops / world / kern_s / 1e12
    traffic, tr_extra = ncu_traffic(5)
    roof = {"bound": "tensor", "kernel": "k_batched_round2<25> (DMMA.8x8x4; TMA chunk ring, one warp per problem octet)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
            "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (fp64 tensor cores)",
            "timing": "CUDA events around every round-kernel launch of the timed solves (on the solve's stream)",
            "kernel_ms_per_round": 1e3 * kern_s / max(1, sum(r.rounds for r in res)),
            "kernel_share_of_step": kern_s / el,
            "whole_call_tflops": flops / el / 1e12,
            "algorithmic_flops_per_round": (10 * 4.0 + 2.0) * m * n * kl,
            "sphere_sweep_tiles": int(sum(r.sphere_sweeps for r in res)),
            "tiles_per_round": int(res[0].tiles)}
    roof.update(tr_extra or {})
    e2e = None
    if not args.no_e2e:
        a_pin = torch.from_numpy(a).pin_memory()
        y_pin = torch.from_numpy(np.ascontiguousarray(Y)).pin_memory()
        x_pin = torch.empty((kl, n), dtype=torch.float64, pin_memory=True)  # the result's host buffer, reused
        e_t, e_it = 0.0, 0
        for s_ in range(args.steps + 1):
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            r = solve_batched(a_pin.to(dev, non_blocking=True), y_pin.to(dev, non_blocking=True), passes=10,
                              rounds=rounds, gap_tol=c["gap_tol"], eta=eta, return_device=False, x_out=x_pin,
                              check_every=every)
            t1.record(stream)
            torch.cuda.synchronize()
            if s_:
                e_t += t0.elapsed_time(t1) / 1000.0
                e_it += r.iterations
        e2e = {"value": e_it * kl * world / e_t, "unit": "rhs-iters/s", "h2d_bytes_per_step": int(a.nbytes + Y.nbytes),
               "d2h_bytes_per_step": int(n * kl * 8 + 5 * kl * 8), "ms_per_step": 1000.0 * e_t / args.steps}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.batched_oracle import batched_apg
        kk = 512
        t0 = time.perf_counter()
        batched_apg(a, np.asarray(Y[:, :kk]), eta=eta, inner_passes=10, rounds=2, gap_tol=1e-300)
        dt = time.perf_counter() - t0
        cores, model = cpu_info()
        cpu = {"value": 20 * kk / dt, "unit": "rhs-iters/s", "cores": blas_threads(), "kind": "port",
               "sample": f"batched oracle (numpy/OpenBLAS GEMMs), {kk} right-hand sides x 2 rounds",
               "cpu_model": model, "nproc": cores}
    r0 = res[0]
    line = {"metric": metric_name(5), "value": its * kl * world / el, "unit": "rhs-iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded bump dictionary + Dirichlet RHS, BASELINE config 5 recipe)",
            "config": {"workload": c["name"], "m": m, "n": n, "k_rhs": K, "solver": "apg (batched)",
                       "inner_passes": 10, "rounds_per_step": rounds, "check_every": every,
                       "parallelism": f"right-hand sides sharded x{world}, no communication",
                       "step": f"{rounds} screened rounds ({10 * rounds} FISTA steps) on every right-hand side"},
            "max_gap": float(r0.gap.max()), "mean_gap": float(r0.gap.mean()),
            "mean_preserved": float(r0.preserved.mean()), "gpu_launches": launches, "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        if not dist.is_initialized():
            if world == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
        if args.config in (3, 4):
            return run_sharded(args, rank, world, dev)
    if args.config == 5:
        return run_batched(args, rank, world, dev)
    from paper_2202_07258_b200 import Problem, SolverConfig, solve

    inst = make_instance(args.config)
    m, n = inst.a.shape
    cfg = SolverConfig(kind=inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol,
                       max_rounds=args.cfg4_rounds if args.config == 4 else None)
    tdt = torch.float32 if inst.a.dtype == np.float32 else torch.float64
    a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).to(dev)  # (n, m) == column-major A
    p_dev = Problem(a_dev.t(), torch.from_numpy(inst.y).to(dev), inst.lower, inst.upper)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        solve(p_dev, cfg, return_device=True)
    torch.cuda.synchronize()
    results = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            results.append(solve(p_dev, cfg, return_device=True))
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    elapsed = ev0.elapsed_time(ev1) / 1000.0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    iters = sum(r.info["iterations"] for r in results)
    launches = sum(r.info["kernel_launches"] for r in results)
    value = world * iters / elapsed  # replicas (configs 1, 2): every rank solves the whole problem
    ms_per_step = 1000.0 * elapsed / args.steps
    conv = all(r.converged for r in results)

    # live roofline of the dominant kernel (one extra, instrumented solve)
    prof_res = solve(p_dev, cfg, return_device=True, profile=True)
    roof = roofline_block(prof_res.info["profile"], args.config)

    # trajectory for the CPU arm (preserved-count bins of this solve)
    bins = k_bins_from_trace(prof_res.info["trace_arrays"], inst.inner_passes)
    if args.write_trajectory and rank == 0:
        os.makedirs(os.path.dirname(traj_path(args.config)), exist_ok=True)
        with open(traj_path(args.config), "w") as fh:
            json.dump({"config": args.config, "k_bins": bins, "rounds": prof_res.rounds,
                       "iterations": prof_res.info["iterations"]}, fh, indent=1)

    # end to end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        p_host = Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=inst.a.dtype, pin=True)
        h2d = p_host.a_matrix.nbytes + 8 * (m + 2 * n)
        e_it, e_t, d2h = 0, 0.0, 0
        e_steps = min(args.steps, args.e2e_steps)
        for s in range(e_steps + 1):
            p_host.release_device()
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            r = solve(p_host, cfg)  # H2D inside, x/theta D2H at the end
            t1.record(stream)
            torch.cuda.synchronize()
            if s == 0:
                continue  # first call warms the pinned path
            e_t += t0.elapsed_time(t1) / 1000.0
            e_it += r.info["iterations"]
            d2h = r.x.nbytes + r.theta.nbytes + 8 * (r.sat_lower.size + r.sat_upper.size)
        p_host.release_device()
        e2e = {"value": world * e_it / e_t, "unit": unit_name(args.config), "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1000.0 * e_t / e_steps, "steps": e_steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores, model = cpu_info()
        bs = reference_module()
        if bs is not None and args.config in (3, 4):
            rate, det = ref_step_rate(bs, inst, bins, args.cpu_budget, kmax=16000 if args.config == 4 else None)
            cpu = {"value": rate, "unit": unit_name(args.config), "cores": blas_threads(), "kind": "reference",
                   "sample": (f"unmodified reference pg_step (solvers.py:101-116, 2 GEMVs per iteration) at "
                              f"{len(bins)} preserved-count bins of this solve, "
                              f"{sum(d['timed_iterations'] for d in det)} iterations, ~{args.cpu_budget:.0f}s"),
                   "cpu_model": model, "nproc": cores}
        elif bs is not None:
            rate, el, rr = ref_solve_rate(bs, inst, True, max_rounds=2000 if args.config == 1 else 100)
            cpu = {"value": rate, "unit": unit_name(args.config), "cores": blas_threads(), "kind": "reference",
                   "sample": (f"unmodified reference solve(), first {rr.rounds} screened rounds "
                              f"({rr.rounds * inst.inner_passes} {STEP_LABEL[inst.kind]}), trace[-1].elapsed"),
                   "cpu_model": model, "nproc": cores}
        else:
            rate, det = cpu_rate(inst, bins, args.cpu_budget)
            cpu = {"value": rate, "unit": unit_name(args.config), "cores": blas_threads(), "kind": "port",
                   "sample": (f"oracle {STEP_LABEL[inst.kind]} at {len(bins)} preserved-count bins of this solve, "
                              f"{sum(d['timed_iterations'] for d in det)} iterations, ~{args.cpu_budget:.0f}s"),
                   "cpu_model": model, "nproc": cores}

    # what screening buys on the GPU (the reference's paired off / on
    # protocol, bench.py:96-115) and, for config 3, BASELINE's stated FISTA
    # restart rule: one solve each, timed with CUDA events
    study = {}
    if rank == 0 and not args.no_study and args.config == 4:
        # BASELINE's PG does not reach a relative gap of 1e-3 in 200,000
        # iterations on this coherent matrix (profiles/r02_cfg4_gap_probe.txt):
        # its step is a fixed round budget.  FISTA on the same shard reaches
        # the fp32 objective tolerance (relative certified gap 1e-4):
        import dataclasses
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r4 = solve(p_dev, dataclasses.replace(cfg, kind="apg", gap_tol=1e-4, relative_gap=True, max_rounds=20000),
                   return_device=True)
        e1.record(stream)
        torch.cuda.synchronize()
        study.update(time_to_rel_gap_1e4_apg_s=e0.elapsed_time(e1) / 1000.0,
                     iterations_rel_gap_1e4_apg=r4.info["iterations"], converged_rel_gap_1e4_apg=r4.converged)
    if rank == 0 and not args.no_study and args.config in (1, 2, 3):
        import dataclasses

        def timed(c, screening=True):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = solve(p_dev, c, screening=screening, return_device=True)
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / 1000.0, r

        t_off, r_off = timed(cfg, screening=False)
        study.update(time_to_gap_unscreened_s=t_off, iterations_unscreened=r_off.info["iterations"],
                     converged_unscreened=r_off.converged,
                     screening_speedup=t_off / (ms_per_step / 1000.0))
        if args.config == 3:
            t_fn, r_fn = timed(dataclasses.replace(cfg, restart="function"))
            study.update(time_to_gap_stated_restart_s=t_fn, iterations_stated_restart=r_fn.info["iterations"],
                         converged_stated_restart=r_fn.converged, certified_gap_stated_restart=r_fn.gap,
                         stated_restart_rule="FISTA restart on an objective increase only (BASELINE config 3)")

    r0 = results[0]
    line = {"metric": metric_name(args.config), "value": value, "unit": unit_name(args.config), "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            # config 3 is one fixed problem (strong scaling when column-sharded over N > 1 ranks, the
            # same word at N = 1 so the per-N lines compare); configs 1-2 do not shard: N replicas
            # (work grows with N: weak), config 4 is weak by construction (a fixed shard per GPU)
            "scaling": "strong" if args.config == 3 else "weak", "vs_baseline": None,
            "replicas": world if (world > 1 and args.config in (1, 2)) else None,
            "dtype": "f32" if inst.a.dtype == np.float32 else "f64",
            "data": "synthetic (seeded numpy, BASELINE config recipe; no public dataset)",
            "config": config_block(args.config, inst),
            "time_to_gap_s": ms_per_step / 1000.0, "converged": conv, "rounds": r0.rounds,
            "iterations_per_solve": r0.info["iterations"], "final_preserved": r0.trace[-1].preserved_count,
            "certified_gap": r0.gap, "gpu_launches": launches, **study, "roofline": roof, "cpu_baseline": cpu,
            "e2e": e2e, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
