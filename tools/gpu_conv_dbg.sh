# conv rows kernel: tests, role timing (debug bit 16), timing
timeout 200 python -m pytest tests/test_cnn_gpu.py -q -x --timeout 60 -p no:cacheprovider 2>&1 | tail -3
for d in 16; do
  echo "debug=$d"; timeout 60 python tools/cnn_bench.py 4 64 24 1 $d 2>&1 | grep conv_rows_prof | sort -u | awk 'NR%4==1' | grep -E 'warp.: (0|1|9),'
done
timeout 60 python tools/cnn_bench.py 4 64 24 10 | cut -c1-400
