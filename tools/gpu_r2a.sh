# round-2 check: GPU suite, smoke, multi-rank relaunch (gloo, two ranks on one GPU)
set -x
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
PB_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --streams 8 --blocks 32 --steps 5 --warmup 3 --skip-cpu --skip-cnn --e2e-steps 1 > gpurun_out/multi2.json 2> gpurun_out/multi2.err; echo rc=$?
tail -c 1500 gpurun_out/multi2.json; tail -20 gpurun_out/multi2.err
