mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 400 --skip-cpu --e2e-steps 0 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; python -c "import json; d=json.load(open('gpurun_out/bench4.json')); print(d['value'], d['roofline']['kernel_ms'])"; tail -3 gpurun_out/bench4.err
timeout 600 python bench.py --no-fuse --steps 200 --skip-cpu --e2e-steps 0 > gpurun_out/bench4_nofuse.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/bench4_nofuse.json')); print(d['value'], d['roofline']['kernel_ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fir_persistent -s 2 -c 1 -o gpurun_out/prof_bank3 python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 > gpurun_out/ncu_bank3.log 2>&1; tail -1 gpurun_out/ncu_bank3.log
