mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputests.log 2>&1; tail -5 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); c=d['cnn']
print('DPD', d['value'], d['roofline']['frac'], d['fir_modes']['exact']['value'], d['fir_modes']['exact']['roofline']['frac'], d['e2e']['value'], d['parity_stream0'], d['clocks'])
print('CNN', c['value'], c['roofline']['frac'], c['e2e']['value'], c['parity_stream0'], c['kernel_ms'])"
bash tools/profile_round.sh 2>&1 | tail -20
