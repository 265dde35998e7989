MG_SELL_TMA=2 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sell_layouts.py -q -m gpu -p no:cacheprovider -x -k "sell or spmv" 2>&1 | tail -2
MG_SELL_TMA=3 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sell_layouts.py -q -m gpu -p no:cacheprovider -x -k "sell or spmv" 2>&1 | tail -2
for v in 0 1 2 3; do echo "== MG_SELL_TMA=$v"; MG_SELL_TMA=$v timeout 300 python tools/kbench.py 3 128 50 2>&1 | grep -E "coarse AMG A_0"; MG_SELL_TMA=$v timeout 300 python tools/apply_bench.py 3 128 50 | grep "us per"; done
