timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2; timeout 300 python tools/path_compare.py 256 512 1024
