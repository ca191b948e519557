timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2_gputest9.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest9.log
tail -4 gpurun_out/r2_gputest9.log
timeout 1500 python bench.py --steps 3 --warmup 1 --no-config4 --skip-cpu --no-sprm-branch > gpurun_out/r2_bench9.json 2> gpurun_out/r2_bench9.err
python -c "import json; d=json.loads(open('gpurun_out/r2_bench9.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ['value','compress_MBps','decompress_MBps','bits_per_base','parity_vs_reference','step_breakdown_ms']})"
timeout 900 python tools/validate_ref_extrapolation.py 16 > gpurun_out/r2_ref_extrap_check.json 2>&1; cat gpurun_out/r2_ref_extrap_check.json
