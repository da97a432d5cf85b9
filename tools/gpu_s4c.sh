mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_slab_newton.py -q > gpurun_out/s4c_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s4c_pytest.log
timeout 600 python tools/slab_graph_probe.py 1024 16 > gpurun_out/s4c_slab_graph.txt 2>&1; echo probe rc=$?
timeout 600 python tools/slab_graph_probe.py 256 4 >> gpurun_out/s4c_slab_graph.txt 2>&1; echo probe2 rc=$?
