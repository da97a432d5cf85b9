mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_lanes.py -m gpu -q 2>&1 | tail -1
for i in 1 2 3; do timeout 300 python tools/bench_batched_probe.py > gpurun_out/p2_$i.log 2>&1; echo probe rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/p2_$i.log').read().strip().splitlines()[-1]); print({k:round(v['pairs_per_s'],1) for k,v in d.items()})" 2>&1 | tail -1; done
for i in 1 2; do timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 8 --batch 8 --passes 3 > gpurun_out/p1.json 2> gpurun_out/p1.err; python -c "import json; print('batch.py', json.load(open('gpurun_out/p1.json'))['pairs_per_s'])"; done
