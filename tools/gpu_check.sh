# verification pass: GPU tests, smoke, bench line (GPU arm)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s3_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s3_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo bench rc=$?
