#!/bin/bash
# bench.py once per library variant: tools/variant_bench.sh base b66 b86 ...
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_1604_02153_b200/libvrg.so; else lib=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so; fi
  VRG_LIB_PATH=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/vb_$v.json 2> gpurun_out/vb_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/vb_{v}.json"))
except Exception as e:
    print(v, "FAILED", e); sys.exit()
ks = {k.split(" ")[0]: round(x["avg_us"], 2) for k, x in d["kernels"].items()}
print(v, round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), ks)
PY
done
