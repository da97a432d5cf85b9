mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s4a_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s4a_pytest.log
for i in 1 2; do timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 8 --batch 8 --passes 3 > gpurun_out/s4a_b5_$i.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/s4a_b5_$i.json')); print('b5', d['pairs_per_s'])" >> gpurun_out/s4a.txt; done
for c in config1 config2_; do timeout 300 python tools/small_solve_probe.py $c 3 >> gpurun_out/s4a.txt 2>&1; done
