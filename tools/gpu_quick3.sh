for v in 1 0; do MG_SPGEMM_ROWWISE=$v timeout 300 python tools/explore_opts.py 3 128 rw$v: ; done
timeout 1200 python -m pytest tests/test_gpu_mgr_gmres.py tests/test_gpu_amg.py tests/test_gpu_kernels.py tests/test_gpu_determinism.py tests/test_golden.py -q -m gpu -p no:cacheprovider -x > gpurun_out/quick_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/quick_tests.log
