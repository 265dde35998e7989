"""Benchmark: solved DOFs/s of MGR-GMRES (fp64, rtol 1e-8) on BASELINE config 3.

One step = one linear system solved end to end on the device: per-cell block
scaling, MGR + AMG setup, GMRES(30) to rtol 1e-8 (SURVEY.md §8(d) metric:
n / (t_setup + t_solve)).  ``value`` is measured with the matrix and rhs
already resident in HBM; ``e2e`` repeats the step through the public API
with host buffers (pinned host -> device upload of A and b, device -> host
read of x inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--edge 128]
    python bench.py --impl reference ...   # CPU oracle port on the host cores

Multi-GPU: replicas only (the solve does not shard); each
rank solves its own system, time = max over ranks, scaling "weak".
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solved DOFs/s (MGR-GMRES fp64, rtol 1e-8)"
UNIT = "DOF/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--edge", type=int, default=None)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-variants", action="store_true",
                   help="skip the R/P-kind side measurements (SURVEY D5) after the timed run")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None
        self.i0 = 0

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def wait_ready(self, timeout=15.0):
        """Block until nvidia-smi has produced its first sample: its start-up
        stalls the driver (tens of ms), which must not land in a timed step."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)
        time.sleep(0.2)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def mark(self):
        """Start of the timed region: only samples from here on are summarised.
        (nvidia-smi is started before the warm-up so that its start-up, which
        briefly stalls the driver, is not inside the timed region.)"""
        self.i0 = len(self.rows)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = list(self.rows[self.i0:]) or list(self.rows)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 7:
                continue
            for k, nm in enumerate(names):
                if r[3 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class NvmlClockSampler:
    """In-process NVML sampling of the same fields (SM clock, max SM clock,
    clock-event reasons) every 200 ms during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, device):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        self.rows = []
        self.i0 = 0
        self.stop_ev = threading.Event()
        self.t = None

    def start(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, mx, rs))
            except Exception:  # noqa: BLE001
                pass
            self.stop_ev.wait(0.2)

    def wait_ready(self, timeout=15.0):
        t0 = time.perf_counter()
        while not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)

    def mark(self):
        self.i0 = len(self.rows)

    def stop(self):
        self.stop_ev.set()
        self.t.join(timeout=2)
        rows = list(self.rows[self.i0:]) or list(self.rows)
        reasons = sorted({nm for _, _, r in rows for bit, nm in self.REASONS.items() if r & bit})
        sm = [float(r[0]) for r in rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][1]) if rows else None,
                "reasons": reasons, "samples": len(sm), "source": "nvml"}


class _NoClocks:
    def start(self):
        pass

    def wait_ready(self):
        pass

    def mark(self):
        pass

    def stop(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["not sampled (BENCH_CLOCKS=off)"]}


def clock_sampler(device):
    kind = os.environ.get("BENCH_CLOCKS", "smi")
    if kind == "off":
        return _NoClocks()
    if kind == "nvml":
        try:
            return NvmlClockSampler(device)
        except Exception:  # noqa: BLE001
            pass
    return ClockSampler(device)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def _oracle_solve(cfg, edge, rtol=1e-8):
    """One oracle solve (oracle/pipeline.py: the reference's MGR + GMRES restated with
    the PMIS / extended+i / L1 AMG in the amg_mod seam), single-threaded; runs in a
    spawned process (test infrastructure: the checker / CPU baseline, never the
    measured GPU path)."""
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    sys.path.insert(0, ROOT)
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # noqa: BLE001
        pass
    from oracle import amg as oamg, mgr as omgr, pipeline as opipe
    from paper_1801_08464_b200 import pipeline as gpipe, synth
    s = synth.make_config(cfg, edge)
    plan = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    t0 = time.perf_counter()
    res, _, tm = opipe.solve_synthetic(s, rel_tol=rtol, plan=plan, amg_opts=oamg.AmgOptions(**gpipe.DEFAULT_AMG))
    return {"n": s.n, "iterations": res.iterations, "converged": bool(res.converged), "edge_s": f"{s.nx}x{s.ny}x{s.nz}",
            "setup_s": tm["setup_s"], "solve_s": tm["solve_s"], "total_s": time.perf_counter() - t0}


class CpuBaseline:
    """The oracle port on ONE host core, one full solve of the bench's own system
    (same config, same size, rtol 1e-8), started in a spawned process before the GPU
    work and collected at the end (it runs concurrently with the GPU timed regions,
    whose clock is the device's; one host core of many)."""

    def __init__(self, config, edge):
        import multiprocessing as mp
        self.config, self.edge = config, edge
        self.pool = mp.get_context("spawn").Pool(1)
        self.fut = self.pool.apply_async(_oracle_solve, (config, edge))

    def result(self):
        try:
            r = self.fut.get(timeout=3600)
        except Exception as e:  # noqa: BLE001
            return {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"failed: {e}"}
        finally:
            self.pool.close()
        edge = r.get("edge_s", self.edge)
        return {"value": r["n"] / r["total_s"], "unit": UNIT, "cores": 1, "kind": "port",
                "same_config": True, "setup_s": round(r["setup_s"], 2), "solve_s": round(r["solve_s"], 2),
                "iterations": r["iterations"],
                "sample": f"one full solve of the bench system (config-{self.config} generator at {edge}, "
                          f"{r['n']} DOFs, rtol 1e-8): setup {r['setup_s']:.1f}s + solve {r['solve_s']:.1f}s, "
                          f"{r['iterations']} GMRES its; oracle port (numpy/scipy + C restatement), 1 thread"}


def _avail_gb():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) / 2**20
    except Exception:  # noqa: BLE001
        pass
    return 16.0


def _mgr_desc(b):
    """The solver options both arms run (pipeline defaults, mirrored in oracle/pipeline.py)."""
    from paper_1801_08464_b200 import pipeline as gp
    order = "coarse correction then F-relaxation (post_smoothing)" if gp.default_post_smoothing(b) \
        else "F-relaxation then coarse correction"
    kind = "NONINJECTIVE" if b == 2 else "INJECTIVE"
    return (f"{b}-level MGR, R/P {kind}, {order}; F-relaxation AMG V(1,1), coarse AMG V(1,1), PMIS / extended+i "
            f"(max_elmts {gp.DEFAULT_AMG['max_elmts']}) / L1-Jacobi, theta {gp.DEFAULT_AMG['strength_theta']}, "
            f"coarse cutoff {gp.DEFAULT_AMG['coarse_size_cutoff']}; GMRES(30)")


def reference_arm(args, ws, rank):
    """--impl reference: the reference's algorithm on the host cores -- the CPU oracle
    port (the reference is pure Python; oracle/pipeline.py restates its MGR + GMRES
    with the AMG in the amg_mod seam) -- on the SAME system as our arm (config,
    edge, rtol 1e-8).  Each step is one full solve of that system, run as independent
    single-threaded processes, as many at once as cores and memory allow (~8 GB RSS
    per 128^3 solve): one full wave of min(K, P) concurrent solves.  Warm-up: one
    small solve per worker (module import and first-call costs), not a full-size
    one.  value = min(K, P) * n / wall."""
    if rank != 0:
        return
    import multiprocessing as mp
    from paper_1801_08464_b200 import synth
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    s = synth.make_config(args.config, args.edge)
    n = s.n
    gb_per = max(0.5, 1.9e-6 * n)  # measured: 7.6 GB max RSS at 128^3 (4.19M DOFs)
    procs = max(1, min(args.steps, ncpu, int(_avail_gb() * 0.8 / gb_per)))
    # one full wave: K solves when K <= P, else P (a second, partial wave would
    # leave cores idle and understate the CPU's throughput; ~2 min at 128^3)
    nsolve = min(args.steps, procs)
    ctxmp = mp.get_context("spawn")
    with ctxmp.Pool(procs) as pool:
        pool.starmap(_oracle_solve, [(args.config, 8)] * procs)  # warm-up (small)
        t0 = time.perf_counter()
        rs = pool.starmap(_oracle_solve, [(args.config, args.edge)] * nsolve)
        el = time.perf_counter() - t0
    value = n * nsolve / el
    its = [r["iterations"] for r in rs]
    edge_s = f"{s.nx}x{s.ny}x{s.nz}"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el / nsolve * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config generator)", "impl": "reference",
            "config": {"workload": f"BASELINE config {args.config}: {edge_s} b={s.b}, {n} DOFs, "
                                   f"GMRES(30)+MGR rtol 1e-8",
                       "dofs": n, "mgr": _mgr_desc(s.b),
                       "parallelism": f"{procs} concurrent single-threaded CPU processes, "
                                                 f"{nsolve} full solves (one wave; --steps {args.steps})"},
            "iterations": its[-1], "converged": all(r["converged"] for r in rs),
            "setup_s_median": statistics.median(r["setup_s"] for r in rs),
            "solve_s_median": statistics.median(r["solve_s"] for r in rs),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": f"{nsolve} full solves of the bench system ({edge_s}, {n} DOFs), "
                                       f"{procs} at a time on {ncpu} host cores; GMRES its {min(its)}-{max(its)}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    from paper_1801_08464_b200.replicas import Replicas
    rep = Replicas("nccl" if args.impl == "ours" else "gloo")
    ws, rank, local = rep.world, rep.rank, rep.local
    if args.impl == "reference":
        reference_arm(args, ws, rank)
        rep.close()
        return

    cpu_job = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu_job = CpuBaseline(args.config, args.edge)

    from paper_1801_08464_b200 import _lib, synth
    from paper_1801_08464_b200.pipeline import SyntheticSolver

    ctx = _lib.ctx(local)
    edge = args.edge
    sysm = synth.make_config(args.config, edge, seed=rep.seed())
    n = sysm.n
    solver = SyntheticSolver(rel_tol=1e-8, restart=30, max_iter=400, ctx=ctx)
    a = solver.upload(sysm)
    # rhs resident in HBM
    b_dev = _lib.P()
    x_dev = _lib.P()
    ctx.call("mg_dev_alloc", 8 * n, _lib.ctypes.byref(b_dev))
    ctx.call("mg_dev_alloc", 8 * n, _lib.ctypes.byref(x_dev))
    rhs = np.ascontiguousarray(sysm.rhs)
    ctx.call("mg_memcpy_h2d", b_dev, _lib.ptr(rhs), 8 * n)
    gopts = solver.gopts.to_c()
    res = _lib.GmresRes()

    walls = [0.0, 0.0]

    def device_step():
        t0 = time.perf_counter()
        solver.setup()
        t1 = time.perf_counter()
        ctx.call("mg_gmres_dev", a.h, solver.hier.h, b_dev, x_dev, _lib.ctypes.byref(gopts), -1.0,
                 _lib.ctypes.byref(res))
        walls[0], walls[1] = 1e3 * (t1 - t0), 1e3 * (time.perf_counter() - t1)

    def barrier():
        ctx.sync()
        rep.barrier()

    clk = clock_sampler(local)
    clk.start()  # before the warm-up: nvidia-smi's start-up stalls the driver briefly
    clk.wait_ready()
    for _ in range(args.warmup):
        device_step()
    barrier()
    # ---- timed region (device-resident inputs) --------------------------------------
    gc.collect()
    gc.disable()  # a collector pass (tens of ms with torch loaded) must not land in a timed step
    clk.mark()
    launches0 = ctx.launches
    its = []
    conv = True
    setup_ms, solve_ms = [], []
    ev = _Events(ctx)
    ev.record_start()
    dbg = os.environ.get("BENCH_DEBUG") == "1"
    for _ in range(args.steps):
        tw = time.perf_counter()
        device_step()
        t = ctx.timing()
        if dbg:
            ctx.sync()
            print(f"step wall {1e3 * (time.perf_counter() - tw):.1f} ms (setup call {walls[0]:.1f}, gmres call "
                  f"{walls[1]:.1f}) setup {t.setup_ms:.1f} solve {t.solve_ms:.1f} "
                  f"dev_bytes {ctx.device_bytes / 2**30:.2f} GiB", file=sys.stderr, flush=True)
        setup_ms.append(t.setup_ms)
        solve_ms.append(t.solve_ms)
        its.append(res.iterations)
        conv &= bool(res.converged)
    ev.record_stop()
    barrier()
    gc.enable()
    total_ms = ev.elapsed_ms()
    clocks = clk.stop()
    launches = ctx.launches - launches0
    total_ms = rep.max(total_ms)
    ms_step = total_ms / args.steps
    value = n * ws / (ms_step / 1e3)

    # ---- per-kernel rooflines: one extra profiled step ------------------------------
    ctx.set_profiling(True)
    device_step()
    t = ctx.timing()
    ctx.set_profiling(False)
    hbm, peak_kind = peaks()
    spmv_gbs = t.spmv_bytes * t.spmv_calls / (t.spmv_ms * 1e-3) / 1e9 if t.spmv_ms else None
    vc_gbs = t.vcycle_bytes * t.vcycle_calls / (t.vcycle_ms * 1e-3) / 1e9 if t.vcycle_ms else None
    k0_gbs = t.k0_bytes * t.k0_calls / (t.k0_ms * 1e-3) / 1e9 if t.k0_ms else None
    traffic = None
    try:  # dram bytes per launch of the same kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "k0_ncu.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        traffic = None
    roofline = {"bound": "hbm", "kernel": "k_sell<4, u8 codes, EpiJacobi>: L1-Jacobi sweep (SELL-32 SpMV with "
                                          "1-byte column codes + fused update) on the coarse-AMG level-0 "
                                          "operator (MGR Schur complement); bytes = the stored format's",
                "achieved": k0_gbs, "peak": hbm, "unit": "GB/s", "frac": (k0_gbs / hbm) if k0_gbs else None,
                "traffic": traffic, "peak_kind": peak_kind, "bytes_per_launch": t.k0_bytes,
                "avg_launch_ms": t.k0_ms / max(t.k0_calls, 1), "launches_timed": int(t.k0_calls)}
    vc_roof = {"bound": "hbm", "kernel": "coarse-grid AMG V(1,1) cycle (composite: sweeps, residual, R/P, coarsest) -- mgr.py:369 -> amg.py:355-367",
               "achieved": vc_gbs, "peak": hbm, "unit": "GB/s", "frac": (vc_gbs / hbm) if vc_gbs else None,
               "bytes_per_launch": t.vcycle_bytes, "avg_launch_ms": t.vcycle_ms / max(t.vcycle_calls, 1)}
    phases = {nm: round(t.phase_ms[k], 3) for k, nm in enumerate(
        ["bcsr_spmv", "coarse_amg", "f_relax_amg", "gmres_ortho", "mgr_transfers", "prescale", "d2h_sync"])}
    fr_gbs = t.frelax_bytes / (t.phase_ms[2] * 1e-3) / 1e9 if t.phase_ms[2] and t.frelax_bytes else None
    fr_roof = {"bound": "hbm", "kernel": "MGR F-relaxation AMG V(1,1) cycle on A_ff (composite: sweeps, residual, "
                                        "R/P, coarsest) -- mgr.py:191-201 -> amg.py:355-367",
               "achieved": fr_gbs, "peak": hbm, "unit": "GB/s", "frac": (fr_gbs / hbm) if fr_gbs else None,
               "bytes_per_launch": t.frelax_bytes / max(t.frelax_calls, 1),
               "avg_launch_ms": t.phase_ms[2] / max(t.frelax_calls, 1), "cycles_timed": int(t.frelax_calls)}
    spmv_roof = {"bound": "hbm", "kernel": "BCSR b=2 SpMV (GMRES operator)", "achieved": spmv_gbs, "peak": hbm,
                 "unit": "GB/s", "frac": (spmv_gbs / hbm) if spmv_gbs else None,
                 "bytes_per_launch": t.spmv_bytes, "avg_launch_ms": t.spmv_ms / max(t.spmv_calls, 1)}

    # ---- e2e through the public API with host buffers --------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = _e2e(ctx, sysm, args, rep, barrier)

    # ---- side measurement (not the headline): the reference schema's other R/P kinds ----
    variants = None
    if rank == 0 and ws == 1 and sysm.b == 2 and not args.no_variants:
        variants = _rp_variants(ctx, sysm, b_dev, x_dev, n)

    cpu = cpu_job.result() if cpu_job is not None else None

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE config generator)",
                "config": {"workload": f"BASELINE config {args.config}: {sysm.nx}x{sysm.ny}x{sysm.nz} b={sysm.b}, "
                                       f"{n} DOFs, GMRES(30)+MGR rtol 1e-8",
                           "dofs": n, "nnzb": sysm.nnzb, "mgr": _mgr_desc(sysm.b),
                           "l2": "inputs larger than L2 (BCSR A ~600 MB at 128^3)",
                           "parallelism": f"replicas x{ws}"},
                "iterations": its[-1], "converged": conv, "setup_ms": statistics.median(setup_ms),
                "solve_ms": statistics.median(solve_ms),
                "roofline": roofline, "roofline_vcycle": vc_roof, "roofline_frelax": fr_roof,
                "roofline_spmv": spmv_roof,
                "solve_phase_ms": phases,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks}
        if variants:
            line["rp_kinds"] = variants
        print(json.dumps(line), flush=True)
    rep.close()


def _rp_variants(ctx, sysm, b_dev, x_dev, n, warm=2, reps=3):
    """SURVEY D5 asks for both R/P kinds on the b = 2 configs.  The headline runs
    RpKind.NONINJECTIVE (the north star's literal R = [-A_cf A_ff^-1, I], P = [-A_ff^-1 A_fc; I]
    with the diagonal of A_ff); this times the same setup + solve step on the same resident
    system with the schema's INJECTIVE (R = [0, I]) and INJECTION (R = [0, I], P = [0; I]) kinds
    (mgr.py:47-51), after the timed region, device events on the library stream."""
    from paper_1801_08464_b200 import _lib
    from paper_1801_08464_b200.mgr import RpKind
    from paper_1801_08464_b200.pipeline import SyntheticSolver
    out = {"note": "side measurement after the timed region; the headline value is the noninjective kind"}
    for kind in (RpKind.INJECTIVE, RpKind.INJECTION):
        sv = SyntheticSolver(rel_tol=1e-8, restart=30, max_iter=400, ctx=ctx, rp=kind)
        a = sv.upload(sysm)
        gopts = sv.gopts.to_c()
        res = _lib.GmresRes()
        ev = _Events(ctx)
        sm, so = [], []
        for r in range(warm + reps):
            if r == warm:
                ctx.sync()
                ev.record_start()
            sv.setup()
            ctx.call("mg_gmres_dev", a.h, sv.hier.h, b_dev, x_dev, _lib.ctypes.byref(gopts), -1.0,
                     _lib.ctypes.byref(res))
            if r >= warm:
                t = ctx.timing()
                sm.append(t.setup_ms)
                so.append(t.solve_ms)
        ev.record_stop()
        ctx.sync()
        ms = ev.elapsed_ms() / reps
        out[kind.value] = {"value": n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "iterations": int(res.iterations),
                           "converged": bool(res.converged), "setup_ms": statistics.median(sm),
                           "solve_ms": statistics.median(so)}
        sv.hier.free()
        sv.hier = None
        a.free()
    return out


class _Events:
    """CUDA events recorded on the library context's stream (mg_timer_start / stop)."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.ms = None

    def record_start(self):
        self.ctx.sync()
        self.ctx.call("mg_timer_start")

    def record_stop(self):
        import ctypes
        v = ctypes.c_double()
        self.ctx.call("mg_timer_stop", ctypes.byref(v))
        self.ms = v.value

    def elapsed_ms(self):
        return self.ms


PIPELINE = os.environ.get("BENCH_E2E_PIPELINE", "1") != "0"


def _e2e(ctx, sysm, args, rep, barrier):
    from paper_1801_08464_b200 import _lib
    from paper_1801_08464_b200.pipeline import SyntheticSolver
    import torch
    # pinned host copies of the step's inputs
    rp = torch.from_numpy(np.ascontiguousarray(sysm.rowptr)).pin_memory().numpy()
    ci = torch.from_numpy(np.ascontiguousarray(sysm.col)).pin_memory().numpy()
    vals = torch.from_numpy(np.ascontiguousarray(sysm.vals)).pin_memory().numpy()
    rhs = torch.from_numpy(np.ascontiguousarray(sysm.rhs)).pin_memory().numpy()
    xh = torch.empty(sysm.n, dtype=torch.float64).pin_memory().numpy()
    solver = SyntheticSolver(rel_tol=1e-8, restart=30, max_iter=400, ctx=ctx)
    gopts = solver.gopts.to_c()
    res = _lib.GmresRes()
    from paper_1801_08464_b200.sparse import DeviceMatrix

    # Time-step pipeline: step k's Jacobian upload is issued on the library's
    # copy stream (mg_mat_upload_bsr_async) while step k-1 is set up and solved;
    # every upload of the K steps is issued inside the timed region.
    pending = [None]

    def upload():
        return DeviceMatrix.from_bsr(rp, ci, vals, ctx=ctx, asynchronous=PIPELINE)

    dbg = os.environ.get("BENCH_DEBUG") == "1"

    def step(prefetch):
        t0 = time.perf_counter()
        a = pending[0] if pending[0] is not None else upload()
        pending[0] = upload() if prefetch else None
        solver.a = a
        t1 = time.perf_counter()
        solver.setup(a, sysm.b, sysm.n_cells)
        t2 = time.perf_counter()
        ctx.call("mg_gmres", a.h, solver.hier.h, _lib.ptr(rhs), _lib.ptr(xh), _lib.ctypes.byref(gopts), -1.0,
                 _lib.ctypes.byref(res))
        t3 = time.perf_counter()
        a.free()
        if dbg:
            t4 = time.perf_counter()
            print(f"  upload {1e3 * (t1 - t0):.1f} setup {1e3 * (t2 - t1):.1f} gmres {1e3 * (t3 - t2):.1f} "
                  f"free {1e3 * (t4 - t3):.1f} ms", file=sys.stderr, flush=True)

    nw = max(1, args.warmup)
    for i in range(nw):  # the pool settles with two matrices alive; nothing pending afterwards
        step(PIPELINE and i + 1 < nw)
    barrier()
    gc.collect()
    gc.disable()
    ev = _Events(ctx)  # device events on the library stream (host copies run on it too)
    ev.record_start()
    for i in range(args.steps):
        tw = time.perf_counter()
        step(PIPELINE and i + 1 < args.steps)
        if dbg:
            print(f"e2e step wall {1e3 * (time.perf_counter() - tw):.1f} ms", file=sys.stderr, flush=True)
    ev.record_stop()
    barrier()
    gc.enable()
    el = rep.max(ev.elapsed_ms())
    ms = el / args.steps
    h2d = rp.nbytes + ci.nbytes + vals.nbytes + rhs.nbytes
    return {"value": sysm.n * rep.world / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(xh.nbytes),
            "upload": "pipelined: step k+1's matrix copied on a second stream during step k" if PIPELINE
            else "synchronous"}


if __name__ == "__main__":
    main()
