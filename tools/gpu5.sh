mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 400 --skip-cpu --e2e-steps 0 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; python -c "import json; d=json.load(open('gpurun_out/bench5.json')); print(d['value'], d['roofline']['kernel_ms'], d['clocks'])"; tail -3 gpurun_out/bench5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fir_persistent -s 2 -c 1 -o gpurun_out/prof_bank4 python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 > gpurun_out/ncu_bank4.log 2>&1; tail -1 gpurun_out/ncu_bank4.log
