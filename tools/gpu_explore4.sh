timeout 900 python tools/explore_opts.py 3 128 v11:pre_sweeps=1,post_sweeps=1 v11gr:pre_sweeps=1,post_sweeps=1,gr=1 v10:pre_sweeps=1,post_sweeps=0 v01:pre_sweeps=0,post_sweeps=1 > gpurun_out/explore4.log 2>&1
timeout 900 python tools/explore_opts.py 4 64 v11:pre_sweeps=1,post_sweeps=1 v11gr:pre_sweeps=1,post_sweeps=1,gr=1 >> gpurun_out/explore4.log 2>&1
timeout 900 python tools/explore_opts.py 4 96 v11:pre_sweeps=1,post_sweeps=1 v11gr:pre_sweeps=1,post_sweeps=1,gr=1 >> gpurun_out/explore4.log 2>&1
timeout 900 python tools/explore_opts.py 2 64 base: v11:pre_sweeps=1,post_sweeps=1 >> gpurun_out/explore4.log 2>&1
cat gpurun_out/explore4.log
