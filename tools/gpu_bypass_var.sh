# bypass region variants: engine tests (default build) + matrices/s per variant
timeout 300 python -m pytest tests/test_engine_gpu.py -q -p no:cacheprovider 2>&1 | tail -1
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  echo "$v $(timeout 300 python tools/bypass_bench.py 1024 1024 30 1 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['matrices_per_s']/1e6),'M/s',d['kernel_ms_per_step'])")"
done
