for v in "" tools/variants/p5.so tools/variants/p4.so; do
 for d in 0 15; do
  echo -n "$v debug=$d "; PB_LIB_PATH=$v timeout 60 python tools/cnn_bench.py 4 64 24 5 $d | python -c "import json,sys;d=json.load(sys.stdin);print({k:round(v,3) for k,v in d['kernel_ms'].items()})"
 done
done
