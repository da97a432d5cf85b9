#!/bin/bash
# Config 5b throughput (64 pairs at 256^2) against the number of concurrent lanes per GPU.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lanes.py -x -q > gpurun_out/lanes_test.log 2>&1
for L in ${LANES:-1 2 3 4 6 8}; do
  timeout 600 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes $L --passes 2 > gpurun_out/lanes_$L.json 2> gpurun_out/lanes_$L.err
done
