"""Oracle self-perturbation envelopes (GMRES iteration counts) for the parity tests.

    python tests/golden/make_envelope.py [--procs P] [--only sweep|full] [--full-cases cfg:edge:rtol,...]

For each case the CPU oracle (oracle/pipeline.py: the reference's MGR + GMRES
restated, PMIS / extended+i / L1 AMG in the amg_mod seam) is run unperturbed and
under its two self-perturbation models (``oracle.pipeline.gmres_synthetic``):
"linear" (fixed random diagonal perturbations of A and M^-1) and "noise" (fresh
per-call rounding-size noise on A·v, M^-1 and the CGS2 coefficients, calibrated
against the measured GPU-vs-oracle differences).  Iteration counts go to
tests/golden/envelope.json; tests/test_gpu_parity_sweep.py and
tests/test_gpu_parity_full.py accept a GPU count in [min - 1, max + 1] of a case's
envelope, which always contains the unperturbed oracle's count (checked again
in the tests against an in-test oracle run).

Sweep cases (config 3 edges 8..20, config 4 edges 5..12, configs 1 / 2 small;
configs 3 / 4 also with the reference's AMG cutoff 50, i.e. deep hierarchies):
4 linear + 48 noise seeds.  BASELINE sizes (configs 1 / 2 at 64, config 3 at
128^3 with rtol 1e-10 and 1e-8, config 4 at 48^3): 4 + 4 seeds (a 128^3 oracle
solve takes ~3-4 min on one core).  Every process is single-threaded.
"""
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "envelope.json")

# (config, edge, rtol, cutoff): cutoff None = pipeline.DEFAULT_AMG's (2000);
# 50 = the reference's AmgOptions default (deep hierarchies at small sizes)
SWEEP = ([(3, e, 1e-10, None) for e in range(8, 21)] + [(4, e, 1e-10, None) for e in range(5, 13)]
         + [(1, 16, 1e-10, None), (1, 24, 1e-10, None), (2, 8, 1e-10, None), (2, 12, 1e-10, None),
            (2, 16, 1e-10, None)]
         + [(1, 32, 1e-10, None), (2, 32, 1e-10, None), (3, 32, 1e-10, None)]
         + [(3, e, 1e-10, 50) for e in range(8, 21)] + [(4, e, 1e-10, 50) for e in range(5, 13)])
FULL = [(1, 64, 1e-10, None), (2, 64, 1e-10, None), (3, 128, 1e-10, None), (3, 128, 1e-8, None),
        (4, 48, 1e-10, None), (3, 64, 1e-8, None), (3, 96, 1e-8, None), (4, 64, 1e-8, None), (4, 96, 1e-8, None)]


def key(cfg, edge, rtol, cut=None):
    return f"config{cfg}_{edge}_rtol{rtol:g}" + (f"_cut{cut}" if cut else "")


def run_chunk(task):
    """One setup, then the listed (mode, seed) solves."""
    cfg, edge, rtol, cut, runs = task
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    sys.path.insert(0, ROOT)
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle import amg as oamg, mgr as omgr, pipeline as opipe
    from paper_1801_08464_b200 import pipeline as gpipe, synth
    s = synth.make_config(cfg, edge)
    plan = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    t0 = time.perf_counter()
    kw = dict(gpipe.DEFAULT_AMG)
    if cut:
        kw["coarse_size_cutoff"] = cut
    state, _ = opipe.setup_synthetic(s, amg_opts=oamg.AmgOptions(**kw), plan=plan)
    out = []
    for mode, seed in runs:
        r = opipe.gmres_synthetic(state, s.rhs, rel_tol=rtol, perturb_seed=seed, mode=mode)
        out.append((mode, seed, r.iterations, bool(r.converged)))
    return cfg, edge, rtol, cut, out, time.perf_counter() - t0


def tasks_for(cases, n_lin, n_noise, chunk):
    runs = [("none", None)] + [("linear", s) for s in range(1, n_lin + 1)] + \
           [("noise", 100 + s) for s in range(1, n_noise + 1)]
    out = []
    for cfg, edge, rtol, cut in cases:
        for i in range(0, len(runs), chunk):
            out.append((cfg, edge, rtol, cut, runs[i:i + chunk]))
    return out


def main():
    procs = int(sys.argv[sys.argv.index("--procs") + 1]) if "--procs" in sys.argv else max(1, (os.cpu_count() or 2) - 1)
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    tasks = []
    if only and ":" in only:  # explicit cfg:edge[:cut] list, sweep seeds
        sel = []
        for c in only.split(","):
            f = c.split(":")
            sel.append((int(f[0]), int(f[1]), 1e-10, int(f[2]) if len(f) > 2 else None))
        tasks += tasks_for(sel, 4, 48, 13)
    if only in (None, "sweep"):
        tasks += tasks_for(SWEEP, 4, 48, 13)
    if only in (None, "full"):
        tasks = tasks_for(FULL, 4, 4, 1) + tasks  # largest first
    if "--full-cases" in sys.argv:  # cfg:edge:rtol,... (a subset of FULL, re-run)
        sel = []
        for c in sys.argv[sys.argv.index("--full-cases") + 1].split(","):
            f = c.split(":")
            sel.append((int(f[0]), int(f[1]), float(f[2]), None))
        tasks = tasks_for(sel, 4, 4, 1) + tasks
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    fresh = set()
    with mp.get_context("spawn").Pool(procs) as pool:
        for cfg, edge, rtol, cut, out, el in pool.imap_unordered(run_chunk, tasks):
            k = key(cfg, edge, rtol, cut)
            if k not in fresh:
                data[k] = {"unperturbed": None, "linear": [], "noise": [], "converged": True,
                           "models": {"linear": "oracle.pipeline.PERTURB_LINEAR (A, M^-1 relative)",
                                      "noise": "oracle.pipeline.PERTURB_NOISE (A, M^-1, CGS2 coefficients)"}}
                fresh.add(k)
            e = data[k]
            for mode, seed, its, conv in out:
                if mode == "none":
                    e["unperturbed"] = its
                else:
                    e[mode].append(its)
                e["converged"] &= conv
            e["oracle_s_per_chunk"] = round(el, 1)
            print(k, out[0][0], [o[2] for o in out], f"{el:.1f}s", flush=True)
            with open(OUT, "w") as f:
                json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
