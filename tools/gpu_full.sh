# round-end style pass: tests, smoke, bench (GPU arm + cpu baseline), reference arm, launch list
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" | head -5
python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
python tools/ncu_matvec.py --steps 1 > gpurun_out/plain.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python tools/ncu_matvec.py --steps 1 > gpurun_out/ncu_l.log 2>&1; echo ncu rc=$?
