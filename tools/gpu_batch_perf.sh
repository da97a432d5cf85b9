# config 5b / 3 throughput: lanes x batch sweep, one batched 5b solve launch list
mkdir -p gpurun_out
for cfg in "1 8" "8 1" "1 16" "2 16" "4 16" "2 32" "1 64" "4 8" "8 8"; do
  set -- $cfg
  timeout 600 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes $1 --batch $2 --passes 2 > gpurun_out/b5_L$1_B$2.json 2> gpurun_out/b5_L$1_B$2.err
  python -c "import json; d=json.load(open('gpurun_out/b5_L$1_B$2.json')); print('5b lanes',$1,'batch',$2, round(d['pairs_per_s'],1), 'pairs/s', sum(r['newton_iterations'] for r in d['results']), sum(r['inner_iterations'] for r in d['results']))" 2>&1 | tail -1
done
for cfg in "4 1" "1 8" "2 4"; do
  set -- $cfg
  timeout 600 python -m paper_1604_02153_b200.batch --n 512 --pairs 8 --nt 16 --lanes $1 --batch $2 --passes 2 > gpurun_out/b3_L$1_B$2.json 2> gpurun_out/b3_L$1_B$2.err
  python -c "import json; d=json.load(open('gpurun_out/b3_L$1_B$2.json')); print('3 lanes',$1,'batch',$2, round(d['pairs_per_s'],2), 'pairs/s', sum(r['newton_iterations'] for r in d['results']))" 2>&1 | tail -1
done
