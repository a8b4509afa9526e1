# conv rows kernel: which role bounds each layer (pb_conv_actor.debug bits:
# 1 no input loads, 2 no epilogue, 4 no MMAs, 8 no TMEM stores, 16 role timing)
for d in 0 1 2 8 11 3 10 4 15; do
  echo -n "debug=$d "; timeout 60 python tools/cnn_bench.py 4 64 24 5 $d | python -c "import json,sys;d=json.load(sys.stdin);print({k:round(v,3) for k,v in d['kernel_ms'].items()})"
done
