timeout 900 python -m pytest tests -m gpu -x -q -k "sprm or prepass or pretrain" 2>&1 | tail -2
run() { echo "== $*"; env "$@" timeout 300 python tools/sprm_timeline.py 400000 2>&1 | grep -E "step period|fwd32|bptt32"; }
run PMKLC_SPRM_FWD_X2=0
run PMKLC_SPRM_FWD_X2=1
