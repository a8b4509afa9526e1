timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"bank_|resolve|eq1|advance|carry" -c 40 --csv --log-file gpurun_out/launch_m.csv python bench.py --steps 3 --warmup 3 --skip-cnn --skip-cpu --e2e-steps 0 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launch_m.csv')) if len(r)>10]
h=rows[0]
iK=h.index('Kernel Name'); iM=h.index('Metric Name'); iV=h.index('Metric Value'); iI=h.index('ID')
d={}
for r in rows[1:]:
    d.setdefault((int(r[iI]), r[iK][:40]),{})[r[iM]]=r[iV]
for k,v in sorted(d.items())[-12:]: print(k, v)
PY
