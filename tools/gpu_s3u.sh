mkdir -p gpurun_out
REPS=50 timeout 300 python tools/sl_step_probe.py 108 208 14 > gpurun_out/s3u_sl.txt 2>&1; echo sl rc=$?
N=4096 REPS=10 timeout 300 python tools/sl_step_probe.py 8 >> gpurun_out/s3u_sl.txt 2>&1; echo sl4096 rc=$?
