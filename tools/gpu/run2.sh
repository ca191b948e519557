set -x
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2_gputest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest2.log
tail -5 gpurun_out/r2_gputest2.log
for i in 1 2; do timeout 300 python tools/prof_sprm.py 1000000; done > gpurun_out/r2_sprm2.log 2>&1
cat gpurun_out/r2_sprm2.log
