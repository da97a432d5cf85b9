"""Time to solution of selected bench registrations (bench.TTS_RUNS names as arguments), with
the library VRG_LIB_PATH points to."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1604_02153_b200 import api

names = sys.argv[1:]
bench.TTS_RUNS = {k: v for k, v in bench.TTS_RUNS.items() if any(n in k for n in names)}
ctx = api.Context(0)
r = bench.time_to_solution(ctx, api, False)
print(json.dumps({k: (round(v["gpu_s"], 3), v["newton_iterations"], v["krylov_iterations"]) for k, v in r.items()}))
