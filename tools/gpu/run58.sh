timeout 900 python -m pytest tests -m gpu -x -q -k "tokenizer" > gpurun_out/r2_gputest58.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest20.log
tail -3 gpurun_out/r2_gputest58.log
timeout 600 python tools/bench_tokenizer.py > gpurun_out/r2_tokenizer_sweep58.jsonl 2>&1; grep '"token_bytes": 2' gpurun_out/r2_tokenizer_sweep58.jsonl | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['s'],d['k'],round(d['frac'],3), d['parity_prefix_ok'])"; tail -1 gpurun_out/r2_tokenizer_sweep58.jsonl
