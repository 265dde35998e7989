set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -40 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log
timeout 1800 bash tools/sanitize.sh > gpurun_out/sanitize_summary.log 2>&1; echo "san rc=$?"; cat gpurun_out/sanitize_summary.log
