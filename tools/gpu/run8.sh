timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2_gputest8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest8.log
tail -5 gpurun_out/r2_gputest8.log
timeout 600 python tools/sprm_timeline.py 400000 2>&1 | grep -v Warn
