timeout 300 python -m pytest tests/test_dpd_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 300 python bench.py --steps 100 --skip-cnn --skip-cpu --e2e-steps 0 --exact > gpurun_out/b_exact.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_exact.json')); r=d['roofline']; print('exact', round(d['value']), round(r['frac'],3), round(r['kernel_ms'],4), d['fir_modes']['exact']['fp32']['frac'])"
