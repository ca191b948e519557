for v in 0 1 2 3; do echo "variant $v"; PMKLC_NT_VARIANT=$v timeout 600 python tools/sprm_timeline.py 400000 2>&1 | grep -E "period|nt_stream|bptt32"; done
