set -x
mkdir -p gpurun_out
nproc; python -c "import os; print('cpu_count', os.cpu_count())"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --skip-cpu --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:filter_bank -s 2 -c 1 -o gpurun_out/prof_bank python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 > gpurun_out/ncu_bank.log 2>&1
tail -3 gpurun_out/ncu_bank.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fir_kernel -s 1 -c 1 -o gpurun_out/prof_fir python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 0 --no-fuse > gpurun_out/ncu_fir.log 2>&1
tail -3 gpurun_out/ncu_fir.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; cat gpurun_out/ref.json; tail -3 gpurun_out/ref.err
timeout 600 python bench.py --no-fuse --steps 100 --skip-cpu --e2e-steps 1 > gpurun_out/bench_nofuse.json 2>&1; cat gpurun_out/bench_nofuse.json
