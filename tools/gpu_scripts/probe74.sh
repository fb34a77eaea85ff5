timeout 1500 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider 2>&1 | tail -15
