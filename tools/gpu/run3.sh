timeout 600 python tools/sprm_timeline.py 400000 > gpurun_out/r2_sprm_tl.log 2>&1
cat gpurun_out/r2_sprm_tl.log
