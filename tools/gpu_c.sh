mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_cnn_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 300 python tools/cnn_bench.py 4 64 24 10 > gpurun_out/cnn_bench.json 2> gpurun_out/cnn_bench.err; cat gpurun_out/cnn_bench.json; tail -5 gpurun_out/cnn_bench.err
