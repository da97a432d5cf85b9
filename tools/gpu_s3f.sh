mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host.py -q -x > gpurun_out/s3f_host.log 2>&1; echo host rc=$?; tail -2 gpurun_out/s3f_host.log
timeout 600 python bench.py --no-cpu-baseline --no-tts > gpurun_out/s3f_bench.json 2> gpurun_out/s3f_bench.err; echo bench rc=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3f_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s3f_pytest.log
