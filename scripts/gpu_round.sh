# round-end style GPU pass: tests, bench lines, launch list, ncu captures (one GPU)
mkdir -p gpurun_out
[ -n "$SKIP_TESTS" ] || { python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
python bench.py --ppb 1 --no-cpu-baseline > gpurun_out/bench_ppb1.json 2> gpurun_out/bench_ppb1.err
python bench.py --workload micro > gpurun_out/bench_micro.json 2> gpurun_out/bench_micro.err
python bench.py --workload large --steps 1 --warmup 1 > gpurun_out/bench_large.json 2> gpurun_out/bench_large.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
# the three fine-level SpMV kernels of one solver iteration (fp64 COCG SpMV, fp32 residual, fp32 smooth + dot)
ncu --set full --import-source on --clock-control none -k regex:"k_nbe_spmv|k_nbe32" --launch-skip 60 --launch-count 3 -o /tmp/spmv_k8 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_spmv.log 2>&1
ncu --set full --clock-control none -k regex:"k_update|k_pupdate" --launch-skip 40 --launch-count 2 -o /tmp/vec_k8 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_vec.log 2>&1
for r in spmv_k8 vec_k8; do ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv; ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv; done
ls -la /tmp/*.ncu-rep gpurun_out > gpurun_out/ls.txt
