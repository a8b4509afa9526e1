timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"fir_persistentILb1ELi3E" -s 3 -c 1 -o gpurun_out/merged python bench.py --steps 4 --warmup 3 --skip-cnn --skip-cpu --e2e-steps 0 > gpurun_out/ncu_merged.log 2>&1
tail -2 gpurun_out/ncu_merged.log
python tools/ncu_summary.py gpurun_out/merged.ncu-rep
