mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3z_b8.csv python tools/solve_profile_batch.py 8 > gpurun_out/s3z_ncu.log 2>&1; echo rc=$?
timeout 600 python -m pytest tests/test_gpu_blas.py -q > gpurun_out/s3z_blas.log 2>&1; echo blas rc=$?; tail -2 gpurun_out/s3z_blas.log
