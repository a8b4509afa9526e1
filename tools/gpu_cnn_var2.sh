# conv timing experiments per variant: C3 kernel times (results not checked)
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  echo "$v $(timeout 60 python tools/cnn_bench.py 4 64 24 20 2>&1 | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print({k:round(v,3) for k,v in d['kernel_ms'].items()})")"
done
