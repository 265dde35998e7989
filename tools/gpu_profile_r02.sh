# round-2 evidence: bench line, ncu launch list of a short bench, ncu --set full of the dominant kernel
timeout 900 python bench.py > gpurun_out/bench_r02.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_r02.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled --kernel-name 'regex:k_sell<(int)4, (int)1, (bool)0, mg::EpiJacobi' --launch-skip 1 --launch-count 1 -o gpurun_out/k0_r02 python tools/apply_bench.py 3 128 2 > gpurun_out/ncu_k0.log 2>&1; echo "ncu k0 rc=$?"
