mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s4s_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s4s_pytest.log
for i in 1 2; do timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 4 --batch 16 --passes 3 > gpurun_out/s4s_b5_$i.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/s4s_b5_$i.json')); print('b5', d['pairs_per_s'])" >> gpurun_out/s4s.txt; done
timeout 300 python tools/tts_only.py config3 config2 config1 >> gpurun_out/s4s.txt 2>/dev/null
