timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | grep -E "Error|error|assert|FAILED|def test|^E " | head -30
