# int8 layer 2: repeated C3 runs (hang / race check) and the CNN tests
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
  timeout 60 python tools/cnn_bench.py 4 64 24 50 > gpurun_out/i8_run$i.txt 2>&1; echo "run $i rc=$? $(tail -c 300 gpurun_out/i8_run$i.txt)"
done
timeout 600 python -m pytest tests/test_cnn_gpu.py tests/test_mixed_gpu.py -q -p no:cacheprovider -s --tb=line 2>&1 | grep -E "worst|passed|failed|Error|error|assert" | tail -8
