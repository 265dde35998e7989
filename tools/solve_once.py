"""Setup + one warm solve at a config (for ncu launch lists of the solve phase).
MG_GRAPHS=0 is recommended under ncu so each kernel is a separate launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402

s = synth.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 3, int(sys.argv[2]) if len(sys.argv) > 2 else 128)
solver = pipeline.SyntheticSolver(rel_tol=1e-8)
solver.upload(s)
solver.setup()
ctx = _lib.ctx()
ctx.sync()
print("MARK solve start", ctx.launches, flush=True)
res = solver.solve(s.rhs)
print("MARK solve end", ctx.launches, res.iterations, flush=True)
