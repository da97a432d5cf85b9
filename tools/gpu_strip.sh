python tools/sl_step_probe.py 9 109 209 12 112 212 4 7 107 207 8 108 208 > gpurun_out/strip_probe.txt 2>&1; echo probe rc=$?
N=2048 python tools/sl_step_probe.py 9 109 209 7 107 207 8 108 208 >> gpurun_out/strip_probe.txt 2>&1
N=4096 python tools/sl_step_probe.py 9 109 209 7 107 207 8 108 208 >> gpurun_out/strip_probe.txt 2>&1
cat gpurun_out/strip_probe.txt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline_parity.py -m gpu -q -x 2>&1 | tail -4
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_iter.json')); print(d['value'], d['sl_interp'], {k:v['avg_us'] for k,v in d['kernels'].items()})"
