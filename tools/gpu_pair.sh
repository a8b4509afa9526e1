export PB_LIB_PATH=tools/variants/pair.so
timeout 120 python -m pytest tests/test_cnn_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3
for i in 1 2; do timeout 120 python tools/cnn_bench.py 4 64 24 10 2>&1 | tail -1 | cut -c1-260; done
unset PB_LIB_PATH
timeout 120 python tools/cnn_bench.py 4 64 24 10 2>&1 | tail -1 | cut -c1-260
