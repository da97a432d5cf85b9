mkdir -p gpurun_out
for v in base stripP base stripP; do
  if [ "$v" = base ]; then lib=$PWD/paper_1604_02153_b200/libvrg.so; else lib=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so; fi
  VRG_LIB_PATH=$lib timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 4 --batch 16 --passes 3 > gpurun_out/s4j_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/s4j_$v.json')); print('$v b5', round(d['pairs_per_s'],1))" >> gpurun_out/s4j.txt
  VRG_LIB_PATH=$lib timeout 300 python -m paper_1604_02153_b200.batch --n 512 --pairs 8 --nt 16 --lanes 4 --batch 2 --passes 3 > gpurun_out/s4j3_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/s4j3_$v.json')); print('$v b3', round(d['pairs_per_s'],2))" >> gpurun_out/s4j.txt
done
