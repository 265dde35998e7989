for m in 32768 60000 150000 600000; do
  echo "== MG_SELL_MIN_ROWS=$m"
  MG_SELL_MIN_ROWS=$m MG_PROF_LEVELS=1 timeout 300 python tools/phases.py 3 128 2>&1 | tail -24
done > gpurun_out/explore5.log 2>&1
cat gpurun_out/explore5.log
