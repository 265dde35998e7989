# final round-2 evidence: tests, smoke, bench line, reference arm, checked build, sweep, ncu launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_final.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_final.log 2>&1; echo "ref rc=$?"; tail -c 800 gpurun_out/ref_final.log
bash tools/checked_tests.sh
timeout 1200 python tools/sweep.py --out gpurun_out/sweep_final.jsonl > gpurun_out/sweep_final.log 2>&1; echo "sweep rc=$?"; cut -c1-160 gpurun_out/sweep_final.jsonl
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-variants > gpurun_out/ncu_final.log 2>&1; echo "ncu list rc=$?"
python tools/launch_sum.py gpurun_out/r02_launches_final.csv > gpurun_out/launches_final_summary.txt 2>&1; head -30 gpurun_out/launches_final_summary.txt
