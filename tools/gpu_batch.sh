# batched-pairs iteration: batch tests first, then the whole GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -q > gpurun_out/pytest_batch.log 2>&1; echo batch rc=$?; grep -E "passed|failed|Error|assert" gpurun_out/pytest_batch.log | head -30
echo skip full
