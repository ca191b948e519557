export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_bigru_rec_fused|k_attn_bwd_row|k_bigru_rec$" -s 2400 -c 3 -o gpurun_out/r2_full_plateau python tools/prof_bench.py > gpurun_out/r2_ncu4.log 2>&1; echo "ncu4 rc=$?"
