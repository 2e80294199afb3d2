timeout 300 python scripts/ibc_probe.py > gpurun_out/ibc_probe3.log 2>&1
ECT_TRACE_SOLVE=1 timeout 600 python scripts/stall_probe.py 1e-12 600 > gpurun_out/stall3.log 2>&1
ECT_AMG_FUSED=0 python bench.py --no-cpu-baseline > gpurun_out/bench4_unfused.json 2> gpurun_out/bench4_unfused.err
python bench.py --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err
python -m pytest tests/test_gpu_krylov.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/gpu_tests7.log 2>&1
