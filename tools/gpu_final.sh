# round-end refresh: GPU suite, smoke, bench line + reference arm, round profiles,
# bypass / motion app numbers
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 300 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
ROUND=r2 bash tools/profile_round.sh 2>&1 | grep -E "^[a-z ]+: "
for f in 1 0; do timeout 300 python tools/motion_bench.py 256 256 30 $f > gpurun_out/motion_$f.json 2>/dev/null; done
for f in 1 0; do timeout 300 python tools/bypass_bench.py 1024 1024 30 $f > gpurun_out/bypass_$f.json 2>/dev/null; done
echo done
