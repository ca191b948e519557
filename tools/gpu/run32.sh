timeout 600 python -m pytest tests -m gpu -x -q -k "sprm or prepass or pretrain" 2>&1 | tail -2
run() { echo "== $*"; env "$@" timeout 300 python tools/sprm_timeline.py 400000 2>&1 | grep -E "step period|bptt32|nt_r1|dx_t|emb_walk"; }
run PMKLC_SPRM_FOLLOW=0
run PMKLC_FOLLOW_AFTER=1
run PMKLC_SPRM_FOLLOW=1
run PMKLC_FOLLOW_BPTT_WARPS=8 PMKLC_FOLLOW_BPTT_RESERVE_KB=120 PMKLC_FOLLOW_NT_WARPS=2 PMKLC_FOLLOW_NT_MIN_KB=116
run PMKLC_FOLLOW_BPTT_WARPS=8 PMKLC_FOLLOW_BPTT_RESERVE_KB=120 PMKLC_FOLLOW_NT_WARPS=4 PMKLC_FOLLOW_NT_MIN_KB=0
