timeout 300 python -m pytest tests/test_cnn_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/cnn_bench.py 4 64 24 10 2>&1 | tail -1; done
