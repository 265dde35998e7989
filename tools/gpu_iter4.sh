timeout 900 python -m pytest tests/test_gpu_mgr_gmres.py tests/test_gpu_sell_layouts.py tests/test_gpu_determinism.py tests/test_physics_dropin.py -m gpu -q -x -p no:cacheprovider > gpurun_out/iter_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/iter_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?"; python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_iter.log') if x.startswith('{')][-1]
d=json.loads(l); print({k:d[k] for k in ('value','ms_per_step','setup_ms','solve_ms','iterations')}); print(d['solve_phase_ms']); print({k:round(d[k]['frac'],3) for k in ('roofline','roofline_vcycle','roofline_frelax','roofline_spmv')}); print(d.get('rp_kinds'))
PY
