timeout 300 python tools/path_compare.py 160 192 224 256 320 384
