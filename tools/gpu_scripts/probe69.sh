timeout 1200 python -m pytest tests/test_gpu_scale.py -q -x -p no:cacheprovider -k "hub or huge" 2>&1 | tail -15
