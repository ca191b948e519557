PMKLC_NT_VARIANT=4 timeout 300 python tools/prof_sprm.py 40000 2>&1 | tail -70
