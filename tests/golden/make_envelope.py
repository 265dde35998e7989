"""Oracle self-perturbation envelopes at the BASELINE configs' stated sizes.

    python tests/golden/make_envelope.py [cfg:edge:rtol ...] [--procs P]

For each case the CPU oracle (oracle/pipeline.py: the reference's MGR + GMRES
restated, PMIS / extended+i / L1 AMG) is run unperturbed and with seeds 1-4 of
its self-perturbation ((I + 1e-15 U_a)·A and (I + 1e-13 U_m)·M^-1 with fixed random
diagonals U, ``oracle.pipeline.gmres_synthetic``).  The iteration counts are written to
tests/golden/envelope.json; tests/test_gpu_parity_full.py checks the GPU's count
against [min - 1, max + 1] of this envelope at sizes too large to rerun the
ensemble inside the GPU test step (one unperturbed oracle run is still made there
for the solution check).  Every process is single-threaded (numpy/scipy sparse
kernels are; BLAS pinned to 1 thread).
"""
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "envelope.json")
SEEDS = (None, 1, 2, 3, 4)
DEFAULT_CASES = ["1:64:1e-10", "2:64:1e-10", "3:128:1e-10", "3:128:1e-8"]


def run_one(task):
    cfg, edge, rtol, seed = task
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
    state, setup_s = opipe.setup_synthetic(s, amg_opts=oamg.AmgOptions(**gpipe.DEFAULT_AMG), plan=plan)
    r = opipe.gmres_synthetic(state, s.rhs, rel_tol=rtol, perturb_seed=seed)
    return dict(cfg=cfg, edge=edge, rtol=rtol, seed=seed, iterations=r.iterations, converged=bool(r.converged),
                relres=r.residual_norm / r.rhs_norm, setup_s=setup_s, total_s=time.perf_counter() - t0)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    procs = 5
    if "--procs" in sys.argv:
        procs = int(sys.argv[sys.argv.index("--procs") + 1])
        args = [a for a in args if a != str(procs)]
    cases = args or DEFAULT_CASES
    tasks = []
    for c in cases:
        cfg, edge, rtol = c.split(":")
        tasks += [(int(cfg), int(edge), float(rtol), sd) for sd in SEEDS]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    with mp.get_context("spawn").Pool(procs) as pool:
        for r in pool.imap(run_one, tasks):
            print(json.dumps(r), flush=True)
            key = f"config{r['cfg']}_{r['edge']}_rtol{r['rtol']:g}"
            e = data.setdefault(key, {"perturb": [1e-15, 1e-13], "seeds": [], "iterations": [],
                                      "converged": []})
            if r["seed"] in e["seeds"]:
                k = e["seeds"].index(r["seed"])
                e["iterations"][k], e["converged"][k] = r["iterations"], r["converged"]
            else:
                e["seeds"].append(r["seed"])
                e["iterations"].append(r["iterations"])
                e["converged"].append(r["converged"])
            e["oracle_s"] = round(r["total_s"], 1)
            with open(OUT, "w") as f:
                json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
