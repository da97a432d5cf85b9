mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3r_cfg1.csv python tools/small_solve_probe.py config1 1 > gpurun_out/s3r_ncu.log 2>&1; echo rc=$?
VRG_TRACE=1 timeout 120 python tools/small_solve_probe.py config1 3 > gpurun_out/s3r_trace1.txt 2>&1
