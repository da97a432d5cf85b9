mkdir -p gpurun_out
for v in base cols3 base cols3; do
  if [ "$v" = base ]; then lib=$PWD/paper_1604_02153_b200/libvrg.so; else lib=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so; fi
  echo "== $v" >> gpurun_out/s4u.txt
  VRG_LIB_PATH=$lib REPS=50 timeout 300 python tools/sl_step_probe.py 4 109 14 >> gpurun_out/s4u.txt 2>&1
done
