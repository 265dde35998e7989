timeout 300 python tools/apply_bench.py 3 128 50 > gpurun_out/apply_bench.log 2>&1; cat gpurun_out/apply_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/apply_launches.csv python tools/apply_bench.py 3 128 3 > gpurun_out/apply_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/apply_ncu.log
