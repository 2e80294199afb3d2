timeout 600 python scripts/stall_probe.py 1e-12 600 > gpurun_out/stall4.log 2>&1
python -m pytest tests/test_gpu_binding.py tests/test_trace.py tests/test_gpu_parity.py tests/test_gpu_krylov.py -m gpu -q -s > gpurun_out/gpu_tests8.log 2>&1
python -m pytest tests/test_gpu_large.py -m gpu -q -s > gpurun_out/gpu_tests9.log 2>&1
