timeout 900 python -m pytest tests -m gpu -x -q -k "sprm or prepass or pretrain" > gpurun_out/r2_gputest26.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest26.log
tail -3 gpurun_out/r2_gputest26.log
timeout 600 python tools/sprm_timeline.py 400000 2>&1 | grep -v Warn
