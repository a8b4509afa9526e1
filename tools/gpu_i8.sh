# int8-limb layer 2: CNN GPU tests, then C3 throughput and role timing in both conv modes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_mixed_gpu.py -q -p no:cacheprovider -s --tb=line 2>&1 | grep -E "worst|passed|failed|Error|error|assert" | tail -15
for m in i8 bf16x3; do
  echo "== $m"
  PB_CONV_MATH=$m timeout 120 python tools/cnn_bench.py 4 64 24 20 2>&1 | tail -1
  for d in ${DEBUGS:-16}; do echo "debug=$d"
    PB_CONV_MATH=$m timeout 60 python tools/cnn_bench.py 4 64 24 1 $d 2>&1 | grep -E 'conv_rows_prof": 32|step_ms' | sort | uniq | awk 'NR%4==1' | cut -c1-300
  done
done
