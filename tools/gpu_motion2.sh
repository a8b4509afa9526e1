# fused motion region: motion tests, then motion_bench fused / unfused
timeout 600 python -m pytest tests/test_motion_gpu.py -q -p no:cacheprovider --tb=short 2>&1 | tail -15
for f in 1 0; do timeout 300 python tools/motion_bench.py 256 256 30 $f > gpurun_out/motion_$f.json 2>gpurun_out/motion_$f.err; echo "fuse=$f rc=$?"; head -c 900 gpurun_out/motion_$f.json; echo; done
