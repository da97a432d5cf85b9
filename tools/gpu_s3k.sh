mkdir -p gpurun_out
timeout 300 python tools/sl_step_probe.py 109 112 107 108 14 > gpurun_out/s3k_sl.txt 2>&1; echo sl rc=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3k_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s3k_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s3k_bench.json 2> gpurun_out/s3k_bench.err; echo bench rc=$?
