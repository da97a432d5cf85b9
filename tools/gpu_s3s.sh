mkdir -p gpurun_out
REPS=50 timeout 300 python tools/sl_step_probe.py 109 112 107 108 8 14 > gpurun_out/s3s_sl.txt 2>&1; echo sl rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline_parity.py -q -x > gpurun_out/s3s_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s3s_pytest.log
