timeout 900 python tools/explore_opts.py 3 128 v11: v01:pre_sweeps=0,post_sweeps=1 v02:pre_sweeps=0,post_sweeps=2 v01c4k:pre_sweeps=0,post_sweeps=1,coarse_size_cutoff=4000 > gpurun_out/explore6.log 2>&1
timeout 900 python tools/explore_opts.py 4 96 v11: v01:pre_sweeps=0,post_sweeps=1 >> gpurun_out/explore6.log 2>&1
timeout 900 python tools/explore_opts.py 2 64 v11: v01:pre_sweeps=0,post_sweeps=1 >> gpurun_out/explore6.log 2>&1
timeout 900 python tools/explore_opts.py 1 64 v11: v01:pre_sweeps=0,post_sweeps=1 >> gpurun_out/explore6.log 2>&1
cat gpurun_out/explore6.log
