mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); print(d['value'], d['e2e']['value'], d['sl_interp']['us_per_step'], d['clocks']); print(json.dumps(d.get('batched_pairs'))); print({k:v['gpu_s'] for k,v in d['time_to_solution'].items()}); print(d['cpu_baseline']['value'])"
