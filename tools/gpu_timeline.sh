MG_TIMELINE=1 timeout 300 python tools/setup_once.py 3 128 3 > gpurun_out/timeline.log 2>&1
MG_PROF_LEVELS=1 timeout 300 python tools/phases.py 3 128 > gpurun_out/phases.log 2>&1
tail -40 gpurun_out/phases.log
