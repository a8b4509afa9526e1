# round-2: GPU suite, default bench line, multi-rank (gloo) bench
set -x
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -25
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 800 gpurun_out/bench.err
PB_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --streams 8 --blocks 32 --steps 5 --warmup 3 --skip-cpu --skip-cnn --skip-k10 --e2e-steps 1 > gpurun_out/multi2.json 2> gpurun_out/multi2.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/multi2.json'));print(d['n_gpus'],d['value'],d['output_gather'])"; tail -5 gpurun_out/multi2.err
