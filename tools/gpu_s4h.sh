mkdir -p gpurun_out
REPS=50 timeout 300 python tools/sl_step_probe.py 1 14 > gpurun_out/s4h_sl.txt 2>&1; echo sl rc=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s4h_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s4h_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-tts > gpurun_out/s4h_bench.json 2> gpurun_out/s4h_bench.err; echo bench rc=$?
