export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sprm_head|k_sprm_fwd32|k_sprm_bptt32|k_gemm_nt_r1" -s 200 -c 4 -o gpurun_out/r2_full_sprm python tools/prof_sprm.py 400000 > gpurun_out/r2_ncu5.log 2>&1; echo "ncu rc=$?"
