mkdir -p gpurun_out
for v in pre7 base pre7 base; do
  if [ "$v" = base ]; then lib=$PWD/paper_1604_02153_b200/libvrg.so; else lib=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so; fi
  echo "== $v" >> gpurun_out/s4r.txt
  VRG_LIB_PATH=$lib timeout 300 python tools/tts_only.py config5a >> gpurun_out/s4r.txt 2>/dev/null
done
