# sweep-count / strength variants of both AMG hierarchies at 128^3 config 3, plus per-level phases
MG_PROF_LEVELS=1 timeout 300 python tools/phases.py 3 128 > gpurun_out/phases.log 2>&1
tail -40 gpurun_out/phases.log
timeout 900 python tools/explore_opts.py 3 128 base: v11:pre_sweeps=1,post_sweeps=1 v12:pre_sweeps=1,post_sweeps=2 v21:pre_sweeps=2,post_sweeps=1 fr01:frpre=0,frpost=1 th5:strength_theta=0.5 me3:max_elmts=3 me6:max_elmts=6 > gpurun_out/explore3.log 2>&1
cat gpurun_out/explore3.log
timeout 600 python tools/explore_opts.py 4 64 base: v11:pre_sweeps=1,post_sweeps=1 fr22:frpre=2,frpost=2 th5:strength_theta=0.5 me8:max_elmts=8 > gpurun_out/explore3c4.log 2>&1
cat gpurun_out/explore3c4.log
