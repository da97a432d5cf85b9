mkdir -p gpurun_out
REPS=30 timeout 300 python tools/sl_step_probe.py 14 14 > gpurun_out/s4p_sl.txt 2>&1; echo sl rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline_parity.py tests/test_gpu_host.py -q > gpurun_out/s4p_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s4p_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-tts > gpurun_out/s4p_bench.json 2> gpurun_out/s4p_bench.err; echo bench rc=$?
