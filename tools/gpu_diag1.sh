python tools/parity_diag.py 3 10 > gpurun_out/diag_3_10.log 2>&1
python tools/gmres_trace.py 3 10 1e-10 > gpurun_out/trace_3_10.log 2>&1
MG_GRAPHS=0 python tools/gmres_trace.py 3 10 1e-10 gpu > gpurun_out/trace_3_10_nographs.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_sweep.py tests/test_gpu_kernels.py tests/test_gpu_mgr_gmres.py -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/sweep.log 2>&1
tail -40 gpurun_out/sweep.log
cat gpurun_out/diag_3_10.log
