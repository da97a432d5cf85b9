mkdir -p gpurun_out
for v in base seed4 base seed4; do
  if [ "$v" = base ]; then lib=$PWD/paper_1604_02153_b200/libvrg.so; else lib=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so; fi
  VRG_LIB_PATH=$lib timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 4 --batch 16 --passes 3 > gpurun_out/s4w_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/s4w_$v.json')); print('$v b5', round(d['pairs_per_s'],1))" >> gpurun_out/s4w.txt
  VRG_LIB_PATH=$lib N=4096 REPS=5 timeout 300 python tools/sl_step_probe.py 14 >> gpurun_out/s4w.txt 2>&1
done
