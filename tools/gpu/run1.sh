set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2_gputest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest1.log
timeout 1500 python bench.py --steps 2 --warmup 1 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_gputest1.log
