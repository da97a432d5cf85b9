# round-end style pass: tests, smoke, bench (GPU arm + cpu baseline), reference arm, launch list
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" | head -5
python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
python tools/ncu_matvec.py --steps 1 > gpurun_out/plain.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python tools/ncu_matvec.py --steps 1 > gpurun_out/ncu_l.log 2>&1; echo ncu rc=$?
# one --set full capture per dominant kernel class (band adjoint, band incstate, column pass)
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_eval_band|k_pf_cols_reg" --launch-skip 2 -c 3 -o gpurun_out/ncu_full_r1b python tools/ncu_matvec.py --steps 1 > gpurun_out/ncu_f.log 2>&1; echo ncu full rc=$?
# first adjoint band launch of the matvec (launch order: 16 incremental-state band launches first)
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_eval_band" --launch-skip 16 -c 1 -o gpurun_out/ncu_full_adj python tools/ncu_matvec.py --steps 1 > gpurun_out/ncu_fa.log 2>&1; echo ncu full adj rc=$?
