# A/B of merged-stencil variants (tools/variants/*.so): DPD parity tests and bench headline per variant
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  echo "== $v: $(timeout 300 python -m pytest tests/test_dpd_gpu.py tests/test_dpd_random_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1)"
  for i in 1 2; do
  timeout 300 python bench.py --skip-cpu --skip-cnn --e2e-steps 0 --steps 200 > gpurun_out/ms_$v.json 2>gpurun_out/ms_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ms_$v.json'));r=d['roofline'];print('$v',round(d['value']),round(r['frac'],4),round(r['kernel_ms'],4),d['ms_per_step'])"
  done
done
unset PB_LIB_PATH
if [ -n "${NCU:-}" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 14 python bench.py --skip-cpu --skip-cnn --e2e-steps 0 --steps 2 --warmup 3 2>&1 | grep -E "^  [<a-z].*\(|duration" | sed 's/(pb_.*//' | paste - - | awk '{print $1, $(NF)}' | head -14
fi
