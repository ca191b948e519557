PMKLC_DEBUG_SYNC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "test_per_step_probabilities_bitwise_golden" 2>&1 | grep -E "PMKLC_DEBUG|passed|failed" | head -5
