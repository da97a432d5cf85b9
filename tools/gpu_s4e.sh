mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_slab_newton.py -q > gpurun_out/s4e_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s4e_pytest.log
timeout 600 python tools/slab_newton.py --mode single --max-outer 6 > gpurun_out/s4e_single.json 2> gpurun_out/s4e_single.err; echo single rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 tools/slab_newton.py --mode slab --max-outer 6 > gpurun_out/s4e_slab.json 2> gpurun_out/s4e_slab.err; echo slab rc=$?
timeout 600 python tools/slab_graph_probe.py 1024 16 > gpurun_out/s4e_slab_graph.txt 2>&1; echo probe rc=$?
