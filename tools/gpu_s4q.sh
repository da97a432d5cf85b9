mkdir -p gpurun_out
python tools/ncu_matvec.py --steps 1 > /dev/null 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4q_l1024.csv python tools/ncu_matvec.py --steps 1 > gpurun_out/s4q_a.log 2>&1; echo a rc=$?
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4q_l4096.csv python tools/ncu_matvec.py --n 4096 --nt 32 --steps 1 > gpurun_out/s4q_b.log 2>&1; echo b rc=$?
