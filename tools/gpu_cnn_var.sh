# A/B of conv build variants (tools/variants/*.so): C3 throughput per variant, twice
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  for i in 1 2; do
    echo "$v $(timeout 60 python tools/cnn_bench.py 4 64 24 30 2>&1 | tail -1 | cut -c1-260)"
  done
done
