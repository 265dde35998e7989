# full GPU test suite + one default bench run (logs under gpurun_out/)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider -rA > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|GPU .* its vs oracle|^FAILED" gpurun_out/gpu_tests.log | tail -20
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 4000 gpurun_out/bench.log
