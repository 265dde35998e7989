"""Per-phase wall time of a warm MGR setup (MG_TRACE=1 prints each phase, synchronising)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MG_TRACE", "1")

from paper_1801_08464_b200 import pipeline, synth  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    edge = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    s = synth.make_config(cfg, edge)
    solver = pipeline.SyntheticSolver(rel_tol=1e-8)
    solver.upload(s)
    for rep in range(2):
        print(f"==== setup {rep}", file=sys.stderr, flush=True)
        solver.setup()


if __name__ == "__main__":
    main()
