export PATH=/usr/local/cuda/bin:$PATH
which compute-sanitizer; ls /usr/local/cuda/bin | grep -i sanit
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k test_per_step_probabilities_bitwise_golden > gpurun_out/san41.log 2>&1; echo rc=$?
grep -E "Invalid|misaligned|at 0x|by thread|Address|=========" gpurun_out/san41.log | head -30
