# conv role timing (CTA 0): normal, skip epilogue loads/stores (2), skip MMAs (4), skip converter fill (1)
for d in 16 18 20 17; do echo "debug=$d"
  timeout 60 python tools/cnn_bench.py 4 64 24 1 $d 2>&1 | grep -E 'conv_rows_prof": 3,|step_ms' | sort | uniq | awk -F'"warp": ' '{split($2,a,","); if (!(a[1] in seen)) {seen[a[1]]=1; print}}' | cut -c1-250
done
