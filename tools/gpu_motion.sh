timeout 600 python -m pytest tests/test_motion_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3
python tools/motion_bench.py 256 256 30 > gpurun_out/motion.json 2>gpurun_out/motion.err; cat gpurun_out/motion.json; tail -3 gpurun_out/motion.err
PB_LIB_PATH=tools/variants/imgold.so python tools/motion_bench.py 256 256 30 2>&1 | cut -c1-300
