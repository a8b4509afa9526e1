timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
python tools/e2e_probe2.py > gpurun_out/e2e_probe.json 2>&1; cat gpurun_out/e2e_probe.json
timeout 600 python bench.py --skip-cpu --skip-cnn --steps 100 --e2e-steps 5 > gpurun_out/b_e2e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_e2e.json'));print('value',d['value'],'e2e',d['e2e'])"
