"""Phase profile (EBL_PHASE_PROF build) of k copies of one C1 env: k = 148 (one CTA per SM, no
contention) vs 1184; heaviest and light env."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

N, H, W, STEPS = 1024, 128, 128, 200
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)


def prof(idx):
    n = len(idx)
    b = eb.Batch(n, H, W)
    b.set_terrain(t.fuel_class[idx], t.elevation[idx], t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed[idx], t.wind_direction[idx])
    eb._lib.check(eb.lib().ebl_batch_set_profiling(b.handle, 1))
    for _ in range(2):
        b.set_state(init[idx])
        b.set_key(0, 0, streams=np.asarray(idx, dtype=np.uint64))
        b.step(STEPS)
    pr = np.zeros((n, 10), np.int64)
    eb._lib.check(eb.lib().ebl_batch_profile(b.handle, pr.ctypes.data))
    fin = b.get_state()
    b.close()
    p = pr.mean(0) / STEPS
    return p, fin


_, fin = prof(np.arange(N))
burned = (fin != 0).reshape(N, -1).sum(1)
order = np.argsort(burned)
for name, e in (("heaviest", order[-1]), ("p90", order[int(0.9 * N)]), ("median", order[N // 2]),
                ("light", order[N // 10])):
    for k in (148, 1184):
        p, _ = prof(np.full(k, e))
        print(f"{name:8s} x{k:4d}: P1 {p[0]:6.0f} (dense {p[4]:5.0f} build {p[5]:5.0f})  P2 {p[1]:6.0f} "
              f"(work {p[6]:5.0f})  active {p[2]:6.1f} cand {p[7]:5.0f}  [build: count {p[8]:5.0f} reserve {p[9]:5.0f}]")
