mkdir -p gpurun_out
for lb in "8 8" "4 16" "8 4" "16 4" "2 32" "4 8" "16 2"; do
  set -- $lb
  timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes $1 --batch $2 --passes 3 > gpurun_out/s4g_$1_$2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/s4g_$1_$2.json')); print('lanes $1 batch $2', round(d['pairs_per_s'],1))" >> gpurun_out/s4g.txt
done
for lb in "2 4" "1 8" "4 2" "8 1"; do
  set -- $lb
  timeout 300 python -m paper_1604_02153_b200.batch --n 512 --pairs 8 --nt 16 --lanes $1 --batch $2 --passes 3 > gpurun_out/s4g3_$1_$2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/s4g3_$1_$2.json')); print('cfg3 lanes $1 batch $2', round(d['pairs_per_s'],2))" >> gpurun_out/s4g.txt
done
