mkdir -p gpurun_out
for v in base strip256 base strip256; do
  if [ "$v" = base ]; then lib=$PWD/paper_1604_02153_b200/libvrg.so; else lib=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so; fi
  echo "== $v" >> gpurun_out/s4x.txt
  VRG_LIB_PATH=$lib N=4096 REPS=5 timeout 300 python tools/sl_step_probe.py 7 8 9 14 >> gpurun_out/s4x.txt 2>&1
done
