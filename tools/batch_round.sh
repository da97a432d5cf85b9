#!/bin/bash
# Configs 3 and 5b on one GPU (lanes) and the reference's newtonSolve on the host threads.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
for L in 1 4 8; do
  timeout 600 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes $L --passes 2 > gpurun_out/b5_lanes_$L.json 2> gpurun_out/b5_lanes_$L.err
done
for L in 1 4; do
  timeout 600 python -m paper_1604_02153_b200.batch --n 512 --pairs 8 --nt 16 --lanes $L --passes 2 > gpurun_out/b3_lanes_$L.json 2> gpurun_out/b3_lanes_$L.err
done
timeout 900 python -m paper_1604_02153_b200.batch --impl reference --n 256 --pairs 16 --nt 16 > gpurun_out/b5_ref.json 2> gpurun_out/b5_ref.err
timeout 1200 python -m paper_1604_02153_b200.batch --impl reference --n 512 --pairs 8 --nt 16 > gpurun_out/b3_ref.json 2> gpurun_out/b3_ref.err
echo done
