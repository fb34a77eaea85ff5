timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_distributed.py -q -x -p no:cacheprovider -m gpu 2>&1 | tail -2
timeout 900 python tools/scale_model.py 2>&1 | cut -c1-330
