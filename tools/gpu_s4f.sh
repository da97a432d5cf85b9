mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s4f_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s4f_pytest.log
