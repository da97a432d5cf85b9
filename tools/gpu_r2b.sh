# round-2 session-2 iteration: full GPU tests, bench, config-5b lanes, one 5b solve launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_iter.json')); print(d['value'], d['e2e']['value'], d['sl_interp']['us_per_step'], d.get('time_to_solution'))" 2>&1 | head -5
for L in 8; do
  timeout 600 python -m paper_1604_02153_b200.batch --n 256 --pairs 64 --nt 16 --lanes $L --passes 2 > gpurun_out/b5_lanes_$L.json 2> gpurun_out/b5_lanes_$L.err; echo b5 rc=$?
done
tail -c 600 gpurun_out/b5_lanes_8.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve5b_launches.csv python tools/solve_profile.py > gpurun_out/solve5b.log 2>&1; echo ncu rc=$?
python - <<'PY'
import csv, collections
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/solve5b_launches.csv') if not l.startswith('==')) if r.get('Metric Name')=='gpu__time_duration.sum']
c=collections.Counter(); t=collections.Counter()
for r in rows:
    u={'ns':1e-3,'nsecond':1e-3,'us':1.0,'usecond':1.0,'ms':1e3,'msecond':1e3}[r['Metric Unit']]
    c[r['Kernel Name'][:90]]+=1; t[r['Kernel Name'][:90]]+=float(r['Metric Value'].replace(',',''))*u
print(len(rows),'launches', sum(t.values())/1e3,'ms')
for k,v in t.most_common(25): print(f"{v:9.1f} us {c[k]:6d} x {k}")
PY
