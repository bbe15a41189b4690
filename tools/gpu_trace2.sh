for c in "c2" "c1" "c1 g2n4 hybrid"; do echo "== $c"; python tools/trace_planner.py $c 2>&1 | grep -v "^  P"; done
python tools/path_compare.py 256 512
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "device_plan or random or many_replicas" 2>&1 | tail -2
