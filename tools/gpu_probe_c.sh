timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 8 --batch 8 --passes 2 > gpurun_out/p1.json 2> gpurun_out/p1.err; echo batchpy rc=$?; python -c "import json; print(json.load(open('gpurun_out/p1.json'))['pairs_per_s'])"
timeout 300 python tools/bench_batched_probe.py > gpurun_out/p2.log 2>&1; echo probe rc=$?; tail -c 400 gpurun_out/p2.log
CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/bench_batched_probe.py > gpurun_out/p3.log 2>&1; echo probe_blocking rc=$?; grep -v "^  File\|^    " gpurun_out/p3.log | tail -5
