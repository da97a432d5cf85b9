# round-2 session-3 profiles: launch list of one matvec, --set full of the band kernels, column pass, SL state step
mkdir -p gpurun_out
python tools/ncu_matvec.py --steps 1 > gpurun_out/s3m_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3m_launches.csv python tools/ncu_matvec.py --steps 1 > gpurun_out/s3m_ncu_l.log 2>&1; echo launches rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_eval_strip" --launch-skip 4 -c 1 -o gpurun_out/s3m_inc python tools/ncu_matvec.py --steps 1 > gpurun_out/s3m_ncu_inc.log 2>&1; echo inc rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_eval_strip" --launch-skip 20 -c 1 -o gpurun_out/s3m_adj python tools/ncu_matvec.py --steps 1 > gpurun_out/s3m_ncu_adj.log 2>&1; echo adj rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_pf_cols_reg" --launch-skip 4 -c 1 -o gpurun_out/s3m_cols python tools/ncu_matvec.py --steps 1 > gpurun_out/s3m_ncu_cols.log 2>&1; echo cols rc=$?
ncu --set full --import-source on --clock-control none -k regex:"k_eval_strip|k_pf_cols_reg" --launch-skip 4 -c 2 -o gpurun_out/s3m_sl python tools/sl_step_probe.py 109 > gpurun_out/s3m_ncu_sl.log 2>&1; echo sl rc=$?
