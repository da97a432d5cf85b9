python -m pytest tests -m gpu -q -x 2>&1 | tail -8
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench rc=$?
python tools/ncu_matvec.py --steps 1 > gpurun_out/plain.log 2>&1 && ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_pf_rows|k_pf_cols|k_evaluate" -c 6 -o gpurun_out/prof_r1a python tools/ncu_matvec.py --steps 1 > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
