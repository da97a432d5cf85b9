# quick iteration: gpu tests + short bench (+ optional ncu of a kernel regex given as $1)
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench rc=$?
tail -2 gpurun_out/bench_iter.err
if [ -n "$1" ]; then
python tools/ncu_matvec.py --steps 1 > gpurun_out/plain.log 2>&1 && ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"$1" -c ${2:-4} -o gpurun_out/prof_iter python tools/ncu_matvec.py --steps 1 > gpurun_out/ncu_iter.log 2>&1; echo ncu rc=$?
fi
