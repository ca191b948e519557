timeout 900 python -m pytest tests -m gpu -x -q -k "tokenizer" > gpurun_out/r2_gputest19.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest19.log
tail -3 gpurun_out/r2_gputest19.log
timeout 600 python tools/bench_tokenizer.py > gpurun_out/r2_tokenizer_sweep.jsonl 2>&1; tail -1 gpurun_out/r2_tokenizer_sweep.jsonl
timeout 900 python bench.py --steps 1 --warmup 1 --no-config4 --skip-cpu --no-sprm-branch > gpurun_out/r2_bench19.json 2> gpurun_out/r2_bench19.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r2_bench19.json').read().strip().splitlines()[-1]); c=d['config2']; print(c['mean_frac_u32'], c['mean_frac_u16']); [print(r) for r in c['results']]"
