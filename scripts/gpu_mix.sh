python bench.py --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err
python bench.py --no-cpu-baseline --steps 6 > gpurun_out/bench5b.json 2> gpurun_out/bench5b.err
ECT_NO_GRAPH=1 python bench.py --no-cpu-baseline --steps 6 > gpurun_out/bench5_nograph.json 2> gpurun_out/bench5_nograph.err
python -m pytest tests/test_gpu_krylov.py tests/test_gpu_parity.py tests/test_gpu_binding.py tests/test_trace.py tests/test_gpu_full.py -m gpu -q > gpurun_out/gpu_tests10.log 2>&1
