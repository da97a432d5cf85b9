VRG_FUSED_BANDS=1 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_precond.py -m gpu -q -x 2>&1 | tail -2
for f in 0 1; do VRG_FUSED_BANDS=$f timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fb$f.json 2>gpurun_out/bench_fb$f.err; done
