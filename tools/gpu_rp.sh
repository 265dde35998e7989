# R/P kind per MGR level (report both for configs 1-3)
timeout 600 python tools/explore_opts.py 3 128 'noninjective:' 'injective:rp=injective' 'injection:rp=injection' > gpurun_out/rp_c3_128.txt 2>&1; cat gpurun_out/rp_c3_128.txt | tail -5
timeout 300 python tools/explore_opts.py 2 64 'noninjective:' 'injective:rp=injective' > gpurun_out/rp_c2_64.txt 2>&1; tail -3 gpurun_out/rp_c2_64.txt
timeout 300 python tools/explore_opts.py 1 64 'noninjective:' 'injective:rp=injective' > gpurun_out/rp_c1_64.txt 2>&1; tail -3 gpurun_out/rp_c1_64.txt
timeout 300 python tools/explore_opts.py 3 192 'noninjective:' 'injective:rp=injective' > gpurun_out/rp_c3_192.txt 2>&1; tail -3 gpurun_out/rp_c3_192.txt
