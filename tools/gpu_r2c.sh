# round-2 refresh after the int8 layer: GPU suite, smoke, bench line, profiles
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 400 gpurun_out/bench.err
ROUND=r2 bash tools/profile_round.sh 2>&1 | grep -v "^-\|^d\|^total"
