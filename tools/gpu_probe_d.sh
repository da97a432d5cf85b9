mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -q 2>&1 | tail -2
for i in 1 2 3; do timeout 300 python tools/bench_batched_probe.py > gpurun_out/p2_$i.log 2>&1; echo probe rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/p2_$i.log').read().strip().splitlines()[-1]); print({k:round(v['pairs_per_s'],1) for k,v in d.items()})" 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
