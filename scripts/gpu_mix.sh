for l in aa0f279 eef3643 f0b2c51 d8b37f9; do ECT_PROBE_LIB=gpurun_libs/libectgpu_$l.so timeout 300 python scripts/ibc_probe.py >> gpurun_out/ibc_probe.log 2>&1; done
timeout 300 python scripts/ibc_probe.py >> gpurun_out/ibc_probe.log 2>&1
python -m pytest tests/test_trace.py -m gpu -x -q -s > gpurun_out/gpu_tests4.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
python bench.py --no-cpu-baseline --ppb 8 > gpurun_out/bench3_ppb8.json 2> gpurun_out/bench3_ppb8.err
ECT_AMG_F32=0 timeout 900 python scripts/cfg4_probe.py > gpurun_out/cfg4_f32off.log 2>&1
