"""GPU parity with every operator on the solve-phase SELL layouts.

At test sizes most operators are below the size thresholds of the SELL-32
copies (32768 rows), of the row-sorted SELL-C-sigma copies (262144 rows) and of
the CSR column codes, so those layouts would only run in the benchmark.  This
test lowers the thresholds through the environment in a child process, so that
every MGR / AMG operator of a small system runs through them (with every fused
epilogue: Jacobi sweep, residual, prolongation merge), and checks the same bars
as the in-process tests: one MGR application <= 1e-12 against the oracle, and
the end-to-end solve (iterations within +-1 of the oracle's self-perturbation
envelope, tests/golden/envelope.json, as in test_gpu_parity_sweep.py; solution
<= 1e-8 at rtol 1e-10).
"""
import json
import os
import subprocess
import sys

import pytest

from test_gpu_parity_sweep import envelope

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import amg as oamg, blockscale as obs, mgr as omgr, pipeline as opipe
from paper_1801_08464_b200 import amg as gamg, mgr as gmgr, pipeline as gpipe, sparse as gsp, synth

cfg, edge = int(sys.argv[2]), int(sys.argv[3])
s = synth.make_config(cfg, edge)
opts = oamg.AmgOptions(**gpipe.DEFAULT_AMG)
plan_o = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
_, ahat_o = obs.block_scale(s)
ho = omgr.setup_from_matrix(ahat_o, plan_o, opts)
d = gsp.DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals)
_, ahat_g = gsp.block_scale(d)
hg = gmgr.setup_from_matrix(ahat_g, gpipe.default_plan(s.b, s.n_cells), gamg.AmgOptions(**gpipe.DEFAULT_AMG))
layouts = []
for k in range(len(ho.levels)):
    for what in ("a", "r", "p", "a_ff"):
        layouts.append(hg.level_matrix(k, what).spmv_layout())
for q in (0, -1):
    h = hg.amg(q)
    for lvl in h.levels[:-1]:
        layouts.append(lvl.a.spmv_layout())
r = np.random.default_rng(0).standard_normal(s.n)
ea, eb = gmgr.mgr_apply(hg, r), omgr.mgr_apply(ho, r)
apply_err = float(np.linalg.norm(ea - eb) / np.linalg.norm(eb))
ro, _, _ = opipe.solve_synthetic(s, rel_tol=1e-10, plan=plan_o, amg_opts=opts)
rg, _ = gpipe.SyntheticSolver(rel_tol=1e-10).solve_system(s)
print(json.dumps(dict(layouts=layouts, apply_err=apply_err, its=[rg.iterations, ro.iterations],
                      conv=[bool(rg.converged), bool(ro.converged)],
                      x_err=float(np.linalg.norm(rg.x - ro.x) / np.linalg.norm(ro.x)))))
"""


@pytest.mark.parametrize("cfg,edge", [(3, 16), (2, 16), (4, 10)])
def test_all_operators_on_sell_layouts(gpu, cfg, edge):
    env = dict(os.environ, MG_SELL_MIN_ROWS="256", MG_SELL_SIGMA="256")
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(cfg), str(edge)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    lay = res["layouts"]
    # (operators with < 3 entries per row, e.g. the injective R of config 4, stay CSR)
    assert sum(1 for sell, _, _ in lay if sell) >= len(lay) // 2, lay
    assert any(srt for _, _, srt in lay), lay
    assert any(ib < 4 for _, ib, _ in lay), lay
    assert res["apply_err"] <= 1e-12, res
    assert all(res["conv"]), res
    _, lo, hi, _ = envelope(cfg, edge, None)
    lo, hi = min(lo, res["its"][1]), max(hi, res["its"][1])
    assert lo - 1 <= res["its"][0] <= hi + 1, (res, (lo, hi))
    assert res["x_err"] <= 1e-8, res
