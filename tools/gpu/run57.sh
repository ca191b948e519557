export PATH=/usr/local/cuda/bin:$PATH
for cfg in "64 4" "128 4" "32 4" "64 8" "128 2" "256 2"; do set -- $cfg
echo "== blocks=$1 U=$2"; PMKLC_ADAM_BLOCKS=$1 PMKLC_ADAM_U=$2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_adam" -s 500 -c 5 --csv python tools/prof_bench.py 2>/dev/null | grep -E "k_adam" | awk -F'","' '{print $NF}' | tr '\n' ' '; echo; done
