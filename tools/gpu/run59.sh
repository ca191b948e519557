timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "random_geometry" 2>&1 | tail -15
