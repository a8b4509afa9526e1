mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 400 --skip-cpu --e2e-steps 3 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; python -c "import json; d=json.load(open('gpurun_out/bench6.json')); print('mixed', d['value'], d['roofline']['kernel_ms'], d['e2e'], d['parity_stream0'])"; tail -3 gpurun_out/bench6.err
PB_FIR_MATH=scalar timeout 600 python bench.py --steps 400 --skip-cpu --e2e-steps 0 > gpurun_out/bench6s.json 2> gpurun_out/bench6s.err; python -c "import json; d=json.load(open('gpurun_out/bench6s.json')); print('scalar', d['value'], d['roofline']['kernel_ms'])"
python - <<'PY'
import time, hashlib, os, numpy as np
from concurrent.futures import ThreadPoolExecutor
x = np.random.default_rng(0).integers(0, 255, 64 * 8 * 1024 * 1024 // 64, dtype=np.uint8)
t=time.perf_counter(); hashlib.sha256(x).hexdigest(); print('sha256 1 core GB/s', x.nbytes/(time.perf_counter()-t)/1e9)
bufs=[np.random.default_rng(i).integers(0,255,8*1024*1024,dtype=np.uint8) for i in range(64)]
for th in (8,16,32):
    with ThreadPoolExecutor(th) as p:
        t=time.perf_counter(); list(p.map(lambda b: hashlib.sha256(b).digest(), bufs)); dt=time.perf_counter()-t
    print('sha256', th, 'threads GB/s', 64*8*1024*1024/dt/1e9)
PY
