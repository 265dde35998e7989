#!/bin/bash
# The compute-sanitizer stand-in (the tool is closed on the GPU pool): the kernel
# unit tests with inter-thread protocols, run against libmgrgpu_checked.so
# (-DMG_BOUNDS_CHECK device-side checks: hash-table probe bounds and key presence,
# sort-list capacity, code-bitmap range, PMIS neighbour range, trisolve
# dependency order + a spin bound), with MG_POOL=off (every buffer an exact-size
# cudaMalloc) -- plus the run-to-run bitwise determinism tests on the product
# build and on the checked build.  Log: gpurun_out/checked_tests.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
log=gpurun_out/checked_tests.log
SEL='spgemm or sell_column_codes or csr_column_codes or sorted_sell or bsell or hierarchy_bitwise or vcycle_matches or negative_rows or poisson_reduction or cpr_gauss_seidel or synthetic_hierarchy_bitwise or build_rp'
{
  echo "=== product build: determinism"
  timeout 900 python -m pytest tests/test_gpu_determinism.py -q -m gpu -p no:cacheprovider
  echo "rc=$?"
  echo "=== checked build (MG_LIB=checked MG_POOL=off): determinism + kernel unit tests"
  MG_LIB=checked MG_POOL=off timeout 1500 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_kernels.py \
    tests/test_gpu_amg.py tests/test_physics_dropin.py tests/test_gpu_mgr_gmres.py -q -m gpu -p no:cacheprovider -k "$SEL or determinism or repeatable or unsorted"
  echo "rc=$?"
  MG_LIB=checked python -c "
import sys; sys.path.insert(0, '.')
from paper_1801_08464_b200 import _lib
L = _lib.load(); print('loaded', L._name)"
} > $log 2>&1
grep -E "rc=|passed|failed|loaded|MG_DCHECK" $log
