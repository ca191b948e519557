export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_nt_r1" -s 20 -c 1 -o gpurun_out/r2_nt_follow python tools/prof_sprm.py 400000 > gpurun_out/r2_ncu6.log 2>&1; echo "ncu rc=$?"
PMKLC_SPRM_FOLLOW=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_nt_r1" -s 20 -c 1 -o gpurun_out/r2_nt_plain python tools/prof_sprm.py 400000 > gpurun_out/r2_ncu7.log 2>&1; echo "ncu rc=$?"
