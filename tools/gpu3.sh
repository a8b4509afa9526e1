mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 400 --skip-cpu --e2e-steps 2 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; cat gpurun_out/bench3.json; tail -3 gpurun_out/bench3.err
timeout 600 python bench.py --no-fuse --steps 200 --skip-cpu --e2e-steps 0 > gpurun_out/bench3_nofuse.json 2>&1; cat gpurun_out/bench3_nofuse.json | head -c 600
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fir_persistent -s 2 -c 1 -o gpurun_out/prof_bank2 python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 > gpurun_out/ncu_bank2.log 2>&1; tail -2 gpurun_out/ncu_bank2.log
