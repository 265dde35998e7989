timeout 600 python -m pytest tests/test_gpu_amg.py tests/test_gpu_mgr_gmres.py -q -m gpu -p no:cacheprovider -k "large_dense or pivoting or diagonal_matrix or single_level or exact or ideal" > gpurun_out/dense_tests.log 2>&1; tail -5 gpurun_out/dense_tests.log
timeout 900 python tools/explore_opts.py 3 128 base: cut1000:coarse_size_cutoff=1000 cut2000:coarse_size_cutoff=2000 cut4000:coarse_size_cutoff=4000 > gpurun_out/explore_cut2.log 2>&1
timeout 600 python tools/explore_opts.py 2 64 base: cut1000:coarse_size_cutoff=1000 cut2000:coarse_size_cutoff=2000 >> gpurun_out/explore_cut2.log 2>&1
cat gpurun_out/explore_cut2.log
