mkdir -p gpurun_out
REPS=50 timeout 300 python tools/sl_step_probe.py 108 208 8 14 > gpurun_out/s3t_sl.txt 2>&1; echo sl rc=$?
N=4096 REPS=10 timeout 300 python tools/sl_step_probe.py 7 8 9 14 >> gpurun_out/s3t_sl.txt 2>&1; echo sl4096 rc=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3t_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s3t_pytest.log
