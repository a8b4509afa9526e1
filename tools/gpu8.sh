timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --skip-cpu > gpurun_out/bench8.json 2> gpurun_out/bench8.err; python -c "
import json; d=json.load(open('gpurun_out/bench8.json')); print(d['value'], d['roofline'], d['fp32'], d['tolerance_mode'], d['e2e']['value'])"; tail -3 gpurun_out/bench8.err
