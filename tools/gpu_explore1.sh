bash tools/checked_tests.sh
timeout 600 python tools/explore_opts.py 3 128 base: cut300:coarse_size_cutoff=300 cut1000:coarse_size_cutoff=1000 cut2000:coarse_size_cutoff=2000 > gpurun_out/explore_cut.log 2>&1
cat gpurun_out/explore_cut.log
timeout 900 python tools/explore_opts.py 4 64 base: gr:gr=1 > gpurun_out/explore_c4.log 2>&1
timeout 900 python tools/explore_opts.py 4 96 base: gr:gr=1 >> gpurun_out/explore_c4.log 2>&1
cat gpurun_out/explore_c4.log
