mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_lanes.py tests/test_gpu_precond.py -q -x > gpurun_out/s3n_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s3n_pytest.log
timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 8 --batch 8 --passes 3 > gpurun_out/s3n_b5.json 2>gpurun_out/s3n_b5.err; echo batch rc=$?
timeout 300 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes 1 --batch 8 --passes 2 > gpurun_out/s3n_b5_l1.json 2>>gpurun_out/s3n_b5.err; echo batch1 rc=$?
python - <<'P'
import json
for f in ['gpurun_out/s3n_b5.json','gpurun_out/s3n_b5_l1.json']:
    d=json.load(open(f)); print(f, d['pairs_per_s'], d['wall_s'])
P
