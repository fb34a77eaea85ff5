timeout 1500 python -m pytest tests/test_cpp_reference.py tests/test_cli.py -q -p no:cacheprovider 2>&1 | tail -2
