# fused motion region variants (tools/variants/*.so): frames/s
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  echo "$v $(timeout 120 python tools/motion_bench.py 256 256 30 1 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['frames_per_s']/1e6),'M/s',d['kernel_ms'])")"
done
timeout 300 python -m pytest tests/test_motion_gpu.py -q -p no:cacheprovider 2>&1 | tail -1
