mkdir -p gpurun_out
REPS=50 timeout 300 python tools/sl_step_probe.py 109 112 107 108 14 > gpurun_out/s3g_sl.txt 2>&1; echo sl rc=$?
timeout 600 python bench.py --no-cpu-baseline --no-tts > gpurun_out/s3g_bench.json 2> gpurun_out/s3g_bench.err; echo bench rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "band or strip or irregular or headline" > gpurun_out/s3g_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s3g_pytest.log
