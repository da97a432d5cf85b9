mkdir -p gpurun_out
nproc > gpurun_out/s3p_probe.txt
for c in config1 config2i config2_; do timeout 300 python tools/small_solve_probe.py $c 4 >> gpurun_out/s3p_probe.txt 2>&1; done
VRG_TRACE=1 timeout 300 python tools/small_solve_probe.py config2i 2 > gpurun_out/s3p_trace2i.txt 2>&1
