mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputests.log 2>&1; tail -30 gpurun_out/gputests.log
timeout 300 python tools/cnn_bench.py 4 64 24 20 > gpurun_out/cnn_bench.json 2> gpurun_out/cnn_bench.err; cat gpurun_out/cnn_bench.json; tail -5 gpurun_out/cnn_bench.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
