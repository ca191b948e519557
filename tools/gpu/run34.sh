timeout 600 python -m pytest tests -m gpu -x -q -k "sprm or prepass" 2>&1 | tail -1
run() { echo "== $*"; env "$@" timeout 300 python tools/sprm_timeline.py 400000 2>&1 | grep -E "step period|transpose|nt_r1"; }
for n in 1 2 5 10; do run PMKLC_TR_SLABS=$n; done
