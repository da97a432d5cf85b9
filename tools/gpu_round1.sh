set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -3 gpurun_out/bench1.err
python tools/ncu_matvec.py --steps 1 > gpurun_out/plain.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python tools/ncu_matvec.py --steps 1 > gpurun_out/ncu1.log 2>&1; echo ncu rc=$?
