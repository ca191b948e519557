timeout 1800 python tools/parity_large.py config4 4 16 > gpurun_out/r2_parity_c4.log 2>&1; tail -3 gpurun_out/r2_parity_c4.log
timeout 1800 python tools/parity_large.py config5 4 16 > gpurun_out/r2_parity_c5.log 2>&1; tail -3 gpurun_out/r2_parity_c5.log
