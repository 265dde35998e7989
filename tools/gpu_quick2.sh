timeout 300 python tools/apply_bench.py 3 128 50
timeout 300 python tools/explore_opts.py 3 128 v11:
timeout 1200 python -m pytest tests/test_gpu_mgr_gmres.py tests/test_gpu_amg.py tests/test_gpu_kernels.py tests/test_gpu_determinism.py tests/test_gpu_sell_layouts.py tests/test_physics_dropin.py tests/test_golden.py -q -m gpu -p no:cacheprovider -x > gpurun_out/quick_tests.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/quick_tests.log
