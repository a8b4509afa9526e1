timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; cat gpurun_out/bench7.json; tail -3 gpurun_out/bench7.err
bash tools/profile_round.sh > gpurun_out/profile.log 2>&1; tail -3 gpurun_out/profile.log
