mkdir -p gpurun_out
for v in prev base prev base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1604_02153_b200/libvrg.so; else lib=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so; fi
  echo "== $v" >> gpurun_out/s3l_tts.txt
  VRG_LIB_PATH=$lib timeout 300 python tools/tts_only.py config5a config3 >> gpurun_out/s3l_tts.txt 2>/dev/null
done
REPS=50 timeout 300 python tools/sl_step_probe.py 109 112 107 108 14 > gpurun_out/s3l_sl.txt 2>&1
