for d in 16 31 27; do echo "debug=$d"
timeout 60 python tools/cnn_bench.py 4 64 24 1 $d 2>&1 | grep conv_rows_prof | sort | uniq | awk 'NR%4==1'
done
