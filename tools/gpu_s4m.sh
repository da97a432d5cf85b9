mkdir -p gpurun_out
timeout 600 python tools/dropin_tts.py > gpurun_out/s4m_dropin.txt 2>&1; echo dropin rc=$?
timeout 1200 python -m pytest tests/test_gpu_dropin.py -q > gpurun_out/s4m_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s4m_pytest.log
