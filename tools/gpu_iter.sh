# iteration check: AMG / MGR / GMRES tests, setup timeline, short bench
timeout 900 python -m pytest tests/test_gpu_amg.py tests/test_gpu_mgr_gmres.py tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/iter_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/iter_tests.log
MG_TIMELINE=1 timeout 300 python tools/setup_once.py 3 128 3 > gpurun_out/timeline.log 2>&1; tail -12 gpurun_out/timeline.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?"; python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_iter.log') if x.startswith('{')][-1]
d=json.loads(l); print({k:d[k] for k in ('value','ms_per_step','setup_ms','solve_ms','iterations')})
PY
