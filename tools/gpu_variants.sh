for v in "" tools/variants/g1e2.so; do
 for d in 0; do
  echo -n "$v debug=$d "; PB_LIB_PATH=$v timeout 60 python tools/cnn_bench.py 4 64 24 10 $d | python -c "import json,sys;d=json.load(sys.stdin);print({k:round(v,3) for k,v in d['kernel_ms'].items()})"
 done
 PB_LIB_PATH=$v timeout 60 python tools/cnn_bench.py 4 64 24 1 16 2>&1 | grep conv_rows_prof | sort | uniq | awk 'NR%4==1' | head -4
done
