timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "k2" 2>&1 | grep -E "passed|failed|FAILED" | head -60
