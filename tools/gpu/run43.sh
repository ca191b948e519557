timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "test_per_step_probabilities_bitwise_golden" 2>&1 | tail -1
