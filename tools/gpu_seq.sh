timeout 300 python -m pytest tests/test_gpu_mgr_gmres.py -m gpu -q -p no:cacheprovider -k "pipelined" 2>&1 | tail -8
timeout 900 python tools/sweep.py --sizes 32 --seq 20 --out gpurun_out/sweep_seq.jsonl 2>&1 | tail -3 | cut -c1-600
