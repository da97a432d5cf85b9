# session-3 final pass: GPU suite, smoke, full bench line, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s4o_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s4o_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/s4o_bench.json 2> gpurun_out/s4o_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s4o_bench_ref.json 2> gpurun_out/s4o_bench_ref.err; echo ref rc=$?
