for m in 0 1 2 3; do VRG_PDL=$m python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pdl$m.json 2>/dev/null; done
