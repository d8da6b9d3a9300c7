"""Does the env -> CTA order matter?  C1 batch kernel time with envs in natural order, sorted by
activity (burned cells) descending / ascending, and in a round-robin interleave of the sorted list
(heaviest envs spread one per SM, assuming the block scheduler deals CTAs to SMs in order)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

N, H, W, STEPS = 1024, 128, 128, 200
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)


def run(idx, reps=6):
    b = eb.Batch(N, H, W)
    b.set_terrain(t.fuel_class[idx], t.elevation[idx], t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed[idx], t.wind_direction[idx])
    ms = []
    for i in range(reps + 1):
        b.set_state(init[idx])
        b.set_key(0, 0, streams=np.asarray(idx, dtype=np.uint64))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        b.step(STEPS)
        b.sync()
        e1.record()
        e1.synchronize()
        if i:
            ms.append(e0.elapsed_time(e1))
    fin = b.get_state()
    b.close()
    return float(np.median(ms)), fin


nat = np.arange(N)
ms, fin = run(nat)
burned = (fin != 0).reshape(N, -1).sum(1)
desc = np.argsort(-burned, kind="stable")
print(f"natural   {ms:.3f} ms")
print(f"desc      {run(desc)[0]:.3f} ms")
print(f"asc       {run(desc[::-1].copy())[0]:.3f} ms")
# heaviest 148 first, each group of 148 in descending order (= desc); and the reverse interleave:
# 8 heaviest consecutive (would share SMs if the scheduler filled SMs in order)
blk = desc.reshape(-1, 8)[:128].T.reshape(-1)  # rank k*128 + j ... spreads ranks differently
print(f"strided   {run(blk)[0]:.3f} ms")
# predictor: wind speed x mean source of burnable fuel
src = t.class_veg[t.fuel_class].reshape(N, -1)
pred = t.wind_speed * 1.0
order_p = np.argsort(-pred, kind="stable")
print(f"by wind   {run(order_p)[0]:.3f} ms  (corr(pred, burned) = {np.corrcoef(pred, burned)[0,1]:.2f})")
