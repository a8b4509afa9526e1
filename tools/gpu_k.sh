timeout 300 python -m pytest tests/test_dpd_gpu.py tests/test_mixed_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 300 python bench.py --steps 100 --skip-cnn --skip-cpu --e2e-steps 0 > gpurun_out/b_d.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_d.json')); r=d['roofline']; print('d', round(d['value']), round(r['frac'],3), round(r['kernel_ms'],4), d['parity_stream0'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bank_plan -c 2 python bench.py --steps 2 --warmup 3 --skip-cnn --skip-cpu --e2e-steps 0 2>&1 | grep -E "duration" | tail -2
