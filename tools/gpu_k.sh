timeout 600 python -m pytest tests -q -x -m gpu -p no:cacheprovider 2>&1 | tail -1
timeout 300 python bench.py --steps 200 --skip-cnn --skip-cpu --e2e-steps 0 > gpurun_out/b_d.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_d.json')); r=d['roofline']; print('d', round(d['value']), d['ms_per_step'], round(r['frac'],3), round(r['kernel_ms'],4))"
