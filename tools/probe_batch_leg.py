"""Why the bench's batched_pairs leg is slower than batch.py: the leg on a fresh context, then
after the time-to-solution registrations on the same context, then on a fresh context again."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1604_02153_b200 import api

which = sys.argv[1:] or ["fresh", "tts", "after_tts", "fresh2"]
ctx = api.Context(0)
for w in which:
    t0 = time.perf_counter()
    if w == "tts":
        bench.time_to_solution(ctx, api, False)
        print("tts done", round(time.perf_counter() - t0, 1), flush=True)
        continue
    c = api.Context(0) if w == "fresh2" else ctx
    r = bench.batched_pairs(c, api)
    print(w, json.dumps({k: (v["pairs_per_s"], v["wall_s"]) for k, v in r.items()}), flush=True)
