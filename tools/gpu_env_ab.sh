# A/B of an engine environment switch on the DPD headline (ENVVAR=name; runs 1 vs 0)
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -1
for v in 1 0; do
  for i in 1 2; do
  env $ENVVAR=$v timeout 300 python bench.py --skip-cpu --skip-cnn --e2e-steps 0 --steps 200 > gpurun_out/env_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/env_$v.json'));r=d['roofline'];print('$ENVVAR=$v',round(d['value']),round(r['frac'],4),round(r['kernel_ms'],4),d['ms_per_step'],d['gpu_launches'])"
  done
done
