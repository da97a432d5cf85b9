mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/s4k_torchrun.json 2> gpurun_out/s4k_torchrun.err; echo torchrun rc=$?
tail -c 400 gpurun_out/s4k_torchrun.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 1 --warmup 1 > gpurun_out/s4k_ref.json 2> gpurun_out/s4k_ref.err; echo ref rc=$?
tail -c 300 gpurun_out/s4k_ref.json
