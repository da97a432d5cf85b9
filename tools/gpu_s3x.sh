mkdir -p gpurun_out
for v in 4cc8990_1 4cc8990 base 4cc8990_1 4cc8990 base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1604_02153_b200/libvrg.so; else lib=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so; fi
  VRG_LIB_PATH=$lib timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 8 --batch 8 --passes 3 > gpurun_out/s3x_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/s3x_$v.json')); print('$v', d['pairs_per_s'])" >> gpurun_out/s3x.txt
done
