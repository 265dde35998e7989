#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the unit tests
# that drive the kernels with shared-memory protocols or cross-block flags:
# hash SpGEMM (spgemm.cu), PMIS rounds + extended+i (amg_setup.cu), the sync-free
# triangular solve (trisolve.cu, CPR Gauss-Seidel F-relaxation), the column-code
# bitmap (spmv.cu k_code_range / k_code_bitmap / k_code_dict).
# Logs: gpurun_out/sanitize_<tool>.log (copied to profiles/ when judged).
# MG_POOL=off makes every device buffer its own cudaMalloc so memcheck sees
# out-of-bounds accesses the caching allocator's slabs would hide.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SEL_K='spgemm or sell_column_codes or csr_column_codes or sorted_sell or bsell'
SEL_A='hierarchy_bitwise or vcycle_matches or negative_rows or poisson_reduction'
SEL_P='cpr_gauss_seidel'
for tool in memcheck racecheck synccheck initcheck; do
  log=gpurun_out/sanitize_${tool}.log
  : > $log
  for spec in "tests/test_gpu_kernels.py|$SEL_K" "tests/test_gpu_amg.py|$SEL_A" "tests/test_physics_dropin.py|$SEL_P"; do
    f=${spec%%|*}; k=${spec#*|}
    echo "=== $tool $f -k '$k'" >> $log
    MG_POOL=off timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      $( [ $tool = memcheck ] && echo --leak-check no ) \
      python -m pytest "$f" -q -x -m gpu -k "$k" -p no:cacheprovider >> $log 2>&1
    echo "rc=$?" >> $log
  done
  grep -E "ERROR SUMMARY|rc=|passed|failed" $log
done
