for m in 8 4 8 4 2; do
  echo "== RPT8_MIN=$m"; PMKLC_NT_RPT8_MIN=$m timeout 600 python bench.py --steps 2 --warmup 1 --no-config4 --skip-cpu --no-sprm-branch 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['parity_vs_reference']['container_identical_to_reference'])"
done
