timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2_gputest13.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest13.log
tail -4 gpurun_out/r2_gputest13.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke13.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke13.log
s=$(date +%s); timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench13.json 2> gpurun_out/r2_bench13.err; echo "bench rc=$? wall=$(( $(date +%s) - s ))"
s=$(date +%s); timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_ref13.json 2> gpurun_out/r2_ref13.err; echo "ref rc=$? wall=$(( $(date +%s) - s ))"
