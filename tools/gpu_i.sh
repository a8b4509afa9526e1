timeout 600 python -m pytest tests/test_dpd_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 200 --skip-cnn --skip-cpu --e2e-steps 2 > gpurun_out/bench_dpd.json 2> gpurun_out/bench_dpd.err; python -c "
import json; d=json.load(open('gpurun_out/bench_dpd.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['fir_modes']['exact']['value'], d['e2e']['value'], d['parity_stream0'])"; tail -3 gpurun_out/bench_dpd.err
