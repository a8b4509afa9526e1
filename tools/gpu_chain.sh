# matmul-chain fusion: engine tests, bypass app fused / unfused
timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_fixtures_gpu.py -q -p no:cacheprovider --tb=short 2>&1 | tail -4
for f in 1 0; do timeout 300 python tools/bypass_bench.py 1024 1024 30 $f > gpurun_out/bypass_$f.json 2>gpurun_out/bypass_$f.err; echo "fuse=$f rc=$?"; head -c 700 gpurun_out/bypass_$f.json; echo; done
