export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gemm_nt$|k_gemm_nt<" -s 300 -c 10 --csv python tools/prof_bench.py 2>/dev/null | grep -E "k_gemm_nt" | awk -F'","' '{print $5, $NF}' | head -12
