for cfg_e in "3 96" "3 160" "2 64" "4 64" "4 96" "1 64"; do
  echo "== config/edge $cfg_e"
  timeout 900 python tools/explore_opts.py $cfg_e c2000: c1000:coarse_size_cutoff=1000 c50:coarse_size_cutoff=50 2>&1 | grep -E "^c"
done
