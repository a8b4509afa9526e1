for v in default st1 st2 m5; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=$PWD/tools/variants/$v.so; fi
  timeout 300 python bench.py --steps 100 --skip-cnn --skip-cpu --e2e-steps 0 > gpurun_out/b_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b_$v.json')); r=d['roofline']; print('$v', round(d['value']), round(r['frac'],3), round(r['kernel_ms'],4))"
done
