mkdir -p gpurun_out
REPS=30 timeout 300 python tools/sl_step_probe.py 13 14 13 14 5 > gpurun_out/s3e_graph.txt 2>&1; echo rc=$?
