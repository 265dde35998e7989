timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|^FAILED|GPU .* its vs oracle" gpurun_out/gpu_tests.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/ref.log
