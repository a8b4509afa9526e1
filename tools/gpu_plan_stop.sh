# planner phase timing: variants that end the planner after phase 1/2/3 (ncu, warm caches)
for v in stop1 stop2 stop3 default; do
  if [ $v = default ]; then unset PB_LIB_PATH; else export PB_LIB_PATH=tools/variants/$v.so; fi
  echo "== $v"
  ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:bank_plan -c 3 python bench.py --skip-cpu --skip-cnn --e2e-steps 0 --steps 2 --warmup 3 2>&1 | grep -E "duration"
done
