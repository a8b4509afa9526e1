for v in default pt4m6 pt4m8 pt8m3 pt16m2; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=$PWD/tools/variants/$v.so; fi
  timeout 300 python bench.py --steps 100 --skip-cnn --skip-cpu --e2e-steps 0 > gpurun_out/b_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b_$v.json')); print('$v', round(d['value']), round(d['roofline']['frac'],3), round(d['tolerance_mode']['value']), round(d['tolerance_mode']['hbm_frac_of_step'],3))"
done
