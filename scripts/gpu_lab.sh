# SpMV lab + configs[4] residual probe + ncu of the current k = 8 SpMV kernels
./scripts/spmv_lab/lab > gpurun_out/lab.log 2>&1
python scripts/cfg4_probe.py > gpurun_out/cfg4_probe.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_nbe_spmv|k_nbe32" --launch-skip 60 --launch-count 3 -o /tmp/spmv_cur -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_spmv_cur.log 2>&1
ncu -i /tmp/spmv_cur.ncu-rep --page raw --csv > gpurun_out/spmv_cur_raw.csv
ncu -i /tmp/spmv_cur.ncu-rep --page details --csv > gpurun_out/spmv_cur_details.csv
