timeout 900 python -m pytest tests/test_physics_dropin.py tests/test_gpu_mgr_gmres.py -q -m gpu -p no:cacheprovider -x > gpurun_out/t9.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t9.log
timeout 600 python tools/explore_opts.py 3 128 v11gr:gr=1 > gpurun_out/gr.log 2>&1; cat gpurun_out/gr.log
for v in 64 32; do echo "== MG_SELL_LONG_AVG=$v"; MG_SELL_LONG_AVG=$v timeout 300 python tools/apply_bench.py 3 128 50; MG_SELL_LONG_AVG=$v timeout 300 python tools/explore_opts.py 3 128 v11:; done > gpurun_out/longavg.log 2>&1; cat gpurun_out/longavg.log
timeout 1500 python tools/config4_sweep.py gpu 8,12,16,24,32,48,64,96 > gpurun_out/c4_gpu.log 2>&1; cat gpurun_out/c4_gpu.log
