mkdir -p gpurun_out
timeout 900 python tools/probe_batch_leg.py > gpurun_out/s3q_batchleg.txt 2>&1; echo probe rc=$?
timeout 900 python bench.py > gpurun_out/s3q_bench.json 2> gpurun_out/s3q_bench.err; echo bench rc=$?
