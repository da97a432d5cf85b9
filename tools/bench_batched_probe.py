"""bench.py's batched-pairs leg on its own (fresh process): python tools/bench_batched_probe.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1604_02153_b200 import api

ctx = api.Context(0)
print(json.dumps(bench.batched_pairs(ctx, api)))
