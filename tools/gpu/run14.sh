export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 36000 -c 400 --csv --log-file gpurun_out/r2_launches_bench_plateau.csv python tools/prof_bench.py > gpurun_out/r2_ncu1.log 2>&1; echo "ncu1 rc=$?"
python tools/launches.py gpurun_out/r2_launches_bench_plateau.csv > gpurun_out/r2_launches_bench_plateau.txt 2>&1; head -25 gpurun_out/r2_launches_bench_plateau.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_bigru_rec_fused|k_attn_bwd_row|k_bigru_rec$" -s 300 -c 3 -o gpurun_out/r2_full_bench python tools/prof_bench.py > gpurun_out/r2_ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 560 --csv --log-file gpurun_out/r2_launches_sprm.csv python tools/prof_sprm.py 1000000 > gpurun_out/r2_ncu3.log 2>&1; echo "ncu3 rc=$?"
python tools/launches.py gpurun_out/r2_launches_sprm.csv > gpurun_out/r2_launches_sprm.txt 2>&1; head -20 gpurun_out/r2_launches_sprm.txt
