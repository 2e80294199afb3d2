timeout 300 python scripts/ibc_probe.py > gpurun_out/ibc_probe2.log 2>&1
ECT_TRACE_SOLVE=1 timeout 600 python scripts/stall_probe.py 1e-12 600 > gpurun_out/stall2.log 2>&1
python -m pytest tests/test_trace.py tests/test_gpu_parity.py -m gpu -x -q -s > gpurun_out/gpu_tests5.log 2>&1
timeout 900 python scripts/cfg4_probe.py > gpurun_out/cfg4_b.log 2>&1
python -m pytest tests/test_gpu_large.py -m gpu -x -q -s > gpurun_out/gpu_tests6.log 2>&1
