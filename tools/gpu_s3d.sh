mkdir -p gpurun_out
timeout 300 python tools/sl_step_probe.py 109 112 107 108 7 8 > gpurun_out/s3d_sl.txt 2>&1; echo sl rc=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3d_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s3d_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-tts > gpurun_out/s3d_bench.json 2> gpurun_out/s3d_bench.err; echo bench rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_eval_strip|k_pf_cols_reg" --launch-skip 4 -c 2 -o gpurun_out/s3d_sl_full python tools/sl_step_probe.py 109 > gpurun_out/s3d_ncu.log 2>&1; echo ncu rc=$?
