python tools/bench_batched_probe.py 2>&1 | tail -1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nocpu.json 2> gpurun_out/bench_nocpu.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_nocpu.json')); print(json.dumps(d['batched_pairs']))"
