timeout 300 python -m pytest tests/test_cnn_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3
for d in 0 3 5 6; do echo "debug=$d"; timeout 300 python tools/cnn_bench.py 4 64 24 10 $d 2>&1 | tail -1; done
