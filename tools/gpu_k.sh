timeout 300 python -m pytest tests/test_dpd_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for v in default; do
  timeout 300 python bench.py --steps 100 --skip-cnn --skip-cpu --e2e-steps 0 > gpurun_out/b_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b_$v.json')); r=d['roofline']; print('$v', round(d['value']), round(r['frac'],3), round(r['kernel_ms'],4))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bank_plan -c 3 python bench.py --steps 2 --warmup 3 --skip-cnn --skip-cpu --e2e-steps 0 2>&1 | grep -E "bank_plan|duration" | tail -4
