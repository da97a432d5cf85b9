# packed departure cells + stream-ordered block cache: tests, SL step pieces, bench, batch-leg probe
mkdir -p gpurun_out
timeout 300 python tools/sl_step_probe.py 109 112 104 107 108 > gpurun_out/s3b_sl.txt 2>&1; echo sl rc=$?
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s3b_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s3b_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s3b_bench.json 2> gpurun_out/s3b_bench.err; echo bench rc=$?
timeout 900 python tools/probe_batch_leg.py > gpurun_out/s3b_batchleg.txt 2>&1; echo probe rc=$?
