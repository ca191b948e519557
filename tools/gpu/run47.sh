export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 36000 -c 400 --csv --log-file gpurun_out/r2_launches_plateau47.csv python tools/prof_bench.py > gpurun_out/ncu47a.log 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_attn_bwd_row|k_attn_fwd_row|k_gemm_nt$" -s 1200 -c 3 -o gpurun_out/r2_full_attn47 python tools/prof_bench.py > gpurun_out/ncu47b.log 2>&1; echo "full rc=$?"
