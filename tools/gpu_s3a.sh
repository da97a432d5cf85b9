mkdir -p gpurun_out
timeout 900 python tools/probe_batch_leg.py > gpurun_out/s3a_batchleg.txt 2>&1; echo probe rc=$?
timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 8 --batch 8 --passes 3 > gpurun_out/s3a_b5.json 2>gpurun_out/s3a_b5.err; echo batch rc=$?
python - <<'P' >> gpurun_out/s3a_batchleg.txt
import json; d=json.load(open('gpurun_out/s3a_b5.json')); print('batch.py', d['pairs_per_s'], d['wall_s'])
P
timeout 300 python tools/sl_step_probe.py 109 112 104 > gpurun_out/s3a_sl.txt 2>&1; echo sl rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_eval_strip|k_pf_cols_reg" --launch-skip 4 -c 2 -o gpurun_out/s3a_sl_full python tools/sl_step_probe.py 109 > gpurun_out/s3a_ncu.log 2>&1; echo ncu rc=$?
