timeout 900 python -m pytest tests -m gpu -x -q -k "sprm or prepass" > gpurun_out/r2_gputest5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest5.log
tail -3 gpurun_out/r2_gputest5.log
timeout 600 python tools/sprm_timeline.py 400000 2>&1 | grep -v Warn
for i in 1 2; do timeout 300 python tools/prof_sprm.py 1000000; done
