"""k copies of one C1 env (rank: heaviest / median / light by burned cells) through one C1-length
launch -- a fixed workload for ncu captures of the per-env critical path.
    python scripts/one_env_copies.py heaviest 148"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

N, H, W, STEPS = 1024, 128, 128, 200
which = sys.argv[1] if len(sys.argv) > 1 else "heaviest"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 148
HEAVIEST, MEDIAN, LIGHT = 338, 809, 760  # C1 env ids (scripts/contention.py ranking)
e = {"heaviest": HEAVIEST, "median": MEDIAN, "light": LIGHT}[which]
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)
idx = np.full(k, e)
b = eb.Batch(k, H, W)
b.set_terrain(t.fuel_class[idx], t.elevation[idx], t.class_veg, t.class_den, 30.0)
b.set_wind(t.wind_speed[idx], t.wind_direction[idx])
for _ in range(4):
    b.set_state(init[idx])
    b.set_key(0, 0, streams=idx.astype(np.uint64))
    b.step(STEPS)
b.sync()
print("ok", which, k)
