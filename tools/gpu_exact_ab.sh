# A/B of the bit-exact bank kernel variants: bench headline in --exact mode
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  echo "== $v: $(timeout 300 python -m pytest tests/test_dpd_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1)"
  timeout 300 python bench.py --exact --skip-cpu --skip-cnn --e2e-steps 0 --steps 100 > gpurun_out/ex_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ex_$v.json'));r=d['roofline'];print('$v',round(d['value']),round(r['frac'],4),round(r['kernel_ms'],4),d['ms_per_step'])"
done
