# round-end style pass (round 2): tests, smoke, bench (GPU arm + cpu baseline + time to solution),
# reference arm, launch list and --set full captures of the dominant matvec kernels
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|^CPU\(s\)" | head -2; ldconfig -p | grep -i fftw3 || echo "no libfftw3"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo ref rc=$?
python tools/ncu_matvec.py --steps 1 > gpurun_out/r2_plain.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python tools/ncu_matvec.py --steps 1 > gpurun_out/r2_ncu_l.log 2>&1; echo ncu launches rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_eval_band|k_pf_cols_reg" --launch-skip 2 -c 3 -o gpurun_out/r2_ncu_full python tools/ncu_matvec.py --steps 1 > gpurun_out/r2_ncu_f.log 2>&1; echo ncu full rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_eval_band" --launch-skip 16 -c 1 -o gpurun_out/r2_ncu_full_adj python tools/ncu_matvec.py --steps 1 > gpurun_out/r2_ncu_fa.log 2>&1; echo ncu full adj rc=$?
