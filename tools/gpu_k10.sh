# K=10 leg per library variant (tools/variants/*.so)
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  for i in 1 2; do
    timeout 300 python bench.py --skip-cpu --skip-cnn --skip-mixed --e2e-steps 0 --steps 100 > gpurun_out/k10_$v.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/k10_$v.json'));k=d['k10'];print('$v', 'K4', round(d['value']), d['ms_per_step'], 'K10', round(k['tolerance']['value']), k['tolerance']['ms_per_step'])"
  done
done
