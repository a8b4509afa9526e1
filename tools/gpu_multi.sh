# multi-rank bench path on one GPU (gloo; NCCL refuses two ranks per device)
PB_BENCH_TRACE=1 PB_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --skip-cpu --cnn-steps 3 --e2e-steps 1 --cnn-e2e-steps 1 ${EXTRA:-} > gpurun_out/multi.json 2> gpurun_out/multi.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/multi.json'));print(d['n_gpus'],d['value'],d['output_gather'],d['e2e']['value'],d['cnn']['value'] if d.get('cnn') else None)"
grep "\[rank" gpurun_out/multi.err
