"""Aggregate throughput of T independent solver contexts on ONE GPU (one host thread,
stream and memory pool each; the replicas-only reading of SURVEY 8(e) applied inside a
GPU).  A single MGR-GMRES step leaves the GPU partly idle (latency-bound setup tails,
small AMG levels), so independent systems overlap.  Side measurement, not the bench line.

    python tools/concurrent_bench.py CFG EDGE T [STEPS]
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402


def main():
    cfg, edge, nthr = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    s = synth.make_config(cfg, edge)
    start = threading.Barrier(nthr + 1)
    done = threading.Barrier(nthr + 1)
    its = [0] * nthr

    def worker(k):
        ctx = _lib.ctx(0)
        sv = pipeline.SyntheticSolver(rel_tol=1e-8, ctx=ctx)
        sv.upload(s)
        for _ in range(2):
            sv.setup()
            sv.solve(s.rhs)
        ctx.sync()
        start.wait()
        for _ in range(steps):
            sv.setup()
            r = sv.solve(s.rhs)
        ctx.sync()
        its[k] = r.iterations
        done.wait()

    th = [threading.Thread(target=worker, args=(k,)) for k in range(nthr)]
    for t in th:
        t.start()
    start.wait()
    t0 = time.perf_counter()
    done.wait()
    dt = time.perf_counter() - t0
    for t in th:
        t.join()
    print(f"config {cfg} {edge}^3: {nthr} concurrent solver contexts x {steps} steps: {dt * 1e3 / steps:.1f} ms per "
          f"round of {nthr}, {nthr * steps * s.n / dt / 1e6:.2f} M DOF/s aggregate, its {its}", flush=True)


if __name__ == "__main__":
    main()
