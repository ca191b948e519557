export PATH=/usr/local/cuda/bin:$PATH
for v in old new; do cp vartest/$v.so paper_2507_12805_b200/lib/libpmklc_b200.so; echo "== $v"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gemm_nt$" -s 500 -c 6 --csv python tools/prof_bench.py 2>/dev/null | grep -E "k_gemm_nt" | awk -F'","' '{print $NF}' | tr '\n' ' '; echo; done
