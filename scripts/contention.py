"""Per-CTA latency vs SM sharing: kernel time of k copies of one env (heaviest / median / light
of the C1 batch) for k = 148 (one CTA per SM) ... 1184 (8 per SM)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

N, H, W, STEPS = 1024, 128, 128, 200
KERNEL = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # ebl kernel id (0 auto, 2 resident, 6 warp)
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)


def run(idx, reps=4):
    n = len(idx)
    b = eb.Batch(n, H, W)
    b.set_terrain(t.fuel_class[idx], t.elevation[idx], t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed[idx], t.wind_direction[idx])
    b.set_kernel(KERNEL)
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


ms, fin = run(np.arange(N))
burned = (fin != 0).reshape(N, -1).sum(1)
order = np.argsort(burned)
print(f"mixed 1024: {ms:.3f} ms")
for name, e in (("heaviest", order[-1]), ("median", order[N // 2]), ("light", order[N // 10])):
    row = []
    for k in (148, 296, 592, 1184):
        row.append(f"{k}:{run(np.full(k, e))[0]:.3f}")
    print(f"{name:8s} env {e}: " + "  ".join(row))
