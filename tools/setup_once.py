"""One cold + one warm MGR setup at config 3 (for ncu captures of setup kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import pipeline, synth  # noqa: E402

s = synth.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 3, int(sys.argv[2]) if len(sys.argv) > 2 else 128)
solver = pipeline.SyntheticSolver(rel_tol=1e-8)
solver.upload(s)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
    solver.setup()
