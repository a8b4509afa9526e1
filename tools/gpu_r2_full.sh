# round-2 full pass: GPU suite, smoke, default bench line, round profiles
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 800 gpurun_out/bench.err
ROUND=r2 bash tools/profile_round.sh
