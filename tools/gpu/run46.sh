PMKLC_DEBUG_SYNC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "test_per_step_probabilities" 2>&1 | grep -E "PMKLC_DEBUG|passed|failed" | head -5
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for wt in 1 0; do
  if [ $wt = 0 ]; then export PMKLC_ATTN_NO_WT=1; else unset PMKLC_ATTN_NO_WT; fi
  echo "== WT=$wt"; timeout 600 python bench.py --steps 2 --warmup 1 --no-config4 --skip-cpu --no-sprm-branch 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['parity_vs_reference'] if 'parity_vs_reference' in d else '')"
done
