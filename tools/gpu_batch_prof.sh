mkdir -p gpurun_out
python tools/solve_profile_batch.py 8 > gpurun_out/solveb.log 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve5b_batch8_launches.csv python tools/solve_profile_batch.py 8 > gpurun_out/solveb_ncu.log 2>&1; echo ncu rc=$?
for cfg in "16 4" "8 16" "16 8" "12 8"; do
  set -- $cfg
  timeout 600 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes $1 --batch $2 --passes 2 > gpurun_out/b5_L$1_B$2.json 2> gpurun_out/b5_L$1_B$2.err
  python -c "import json; d=json.load(open('gpurun_out/b5_L$1_B$2.json')); print('5b lanes',$1,'batch',$2, round(d['pairs_per_s'],1), 'pairs/s')" 2>&1 | tail -1
done
