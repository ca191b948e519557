timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2_gputest56.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest56.log
tail -4 gpurun_out/r2_gputest56.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke56.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke56.log
s=$(date +%s); timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench56.json 2> gpurun_out/r2_bench56.err; echo "bench rc=$? wall=$(( $(date +%s) - s ))"
