# CNN tests (single + CTA-pair parity) and the CNN step with / without PB_CONV_PAIR
timeout 300 python -m pytest tests/test_cnn_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
for v in 0 1; do for i in 1 2; do PB_CONV_PAIR=$v timeout 120 python tools/cnn_bench.py 4 64 24 10 2>&1 | tail -1 | cut -c1-230; done; done
