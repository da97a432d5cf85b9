# round-2 iteration: full GPU test suite + a short bench (+ optional ncu launch list)
mkdir -p gpurun_out
nproc; ldconfig -p | grep -i fftw3 || echo "no libfftw3 on this host"
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:--x} > gpurun_out/pytest_r2.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_r2.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench rc=$?
tail -3 gpurun_out/bench_r2.err
