timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --steps 2 --warmup 1 --no-config4 --skip-cpu --no-sprm-branch 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['parity_vs_reference']['container_identical_to_reference'])"; done
