# session-3 final profiles: full bench line, reference arm, matvec launch list, ncu --set full of the band kernels
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/s4b_bench.json 2> gpurun_out/s4b_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s4b_bench_ref.json 2> gpurun_out/s4b_bench_ref.err; echo ref rc=$?
python tools/ncu_matvec.py --steps 1 > gpurun_out/s4b_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4b_launches.csv python tools/ncu_matvec.py --steps 1 > gpurun_out/s4b_ncu_l.log 2>&1; echo launches rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_eval_strip" --launch-skip 4 -c 1 -o gpurun_out/s4b_inc python tools/ncu_matvec.py --steps 1 > gpurun_out/s4b_ncu_inc.log 2>&1; echo inc rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_eval_strip" --launch-skip 20 -c 1 -o gpurun_out/s4b_adj python tools/ncu_matvec.py --steps 1 > gpurun_out/s4b_ncu_adj.log 2>&1; echo adj rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_pf_cols_reg" --launch-skip 4 -c 1 -o gpurun_out/s4b_cols python tools/ncu_matvec.py --steps 1 > gpurun_out/s4b_ncu_cols.log 2>&1; echo cols rc=$?
ncu --set full --import-source on --clock-control none -k regex:"k_eval_strip|k_pf_cols_reg" --launch-skip 4 -c 2 -o gpurun_out/s4b_sl python tools/sl_step_probe.py 109 > gpurun_out/s4b_ncu_sl.log 2>&1; echo sl rc=$?
