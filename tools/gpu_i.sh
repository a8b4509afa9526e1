timeout 600 python -m pytest tests/test_dpd_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 100 --skip-cnn --skip-cpu --e2e-steps 1 > gpurun_out/bench_dpd.json 2> gpurun_out/bench_dpd.err; python -c "
import json; d=json.load(open('gpurun_out/bench_dpd.json')); print(d['value'], d['roofline']['frac'], json.dumps(d['tolerance_mode']))"; tail -3 gpurun_out/bench_dpd.err
