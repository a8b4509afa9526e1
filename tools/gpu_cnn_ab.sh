# A/B of conv kernel variants (tools/variants/*.so): CNN GPU tests + tools/cnn_bench.py
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  echo "== $v: $(timeout 300 python -m pytest tests/test_cnn_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1)"
  for i in 1 2; do timeout 300 python tools/cnn_bench.py 4 64 24 10 2>&1 | tail -1; done
done
