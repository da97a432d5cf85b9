python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for v in L4 L16; do
  VRG_LIB_PATH=$PWD/paper_1604_02153_b200/variants/libvrg_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$v.json 2>/dev/null
done
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_L8.json 2>/dev/null
