"""Per-env phase profile (needs a -DEBL_PHASE_PROF=1 build: scripts/build_variant.sh prof
-DEBL_PHASE_PROF=1, then EBL_LIB=ab/prof.so) of the resident blocked kernel on the C1 batch (ebl_batch_set_profiling):
cycles per step spent in P1 (dense pass + list build) and P2 (sparse decisions), per env, for the
heaviest / p90 / median / lightest envs.  The kernel time is set by the slowest CTA."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

N, H, W, STEPS = 1024, 128, 128, 200
kernel = int(sys.argv[1]) if len(sys.argv) > 1 else 0
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)
b = eb.Batch(N, H, W)
b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
b.set_wind(t.wind_speed, t.wind_direction)
b.set_kernel(kernel)
for prof in (0, 1):
    eb._lib.check(eb.lib().ebl_batch_set_profiling(b.handle, prof))
    ms = []
    for i in range(5):
        b.set_state(init)
        b.set_key(0, 0, first_stream=0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        b.step(STEPS)
        b.sync()
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(f"profiling={prof}: kernel {np.median(ms[1:]):.3f} ms (median of 4)")
pr = np.zeros((N, 10), np.int64)
eb._lib.check(eb.lib().ebl_batch_profile(b.handle, pr.ctypes.data))
p1, p2, act = pr[:, 0] / STEPS, pr[:, 1] / STEPS, pr[:, 2] / STEPS
dense, build, work, cand = pr[:, 4] / STEPS, pr[:, 5] / STEPS, pr[:, 6] / STEPS, pr[:, 7] / STEPS
tot = p1 + p2
order = np.argsort(tot)
print(f"cycles/step: total min {tot.min():.0f} median {np.median(tot):.0f} max {tot.max():.0f}")
for name, e in (("slowest", order[-1]), ("p99", order[int(0.99 * N)]), ("p90", order[int(0.9 * N)]),
                ("median", order[N // 2]), ("fastest", order[0])):
    print(f"{name:8s} env {e:4d}: P1 {p1[e]:6.0f} (dense {dense[e]:5.0f} build {build[e]:5.0f})  "
          f"P2 {p2[e]:6.0f} (work {work[e]:5.0f})  cycles/step; active/step {act[e]:6.1f} cand/step {cand[e]:6.1f}")
# regression of per-step cycles on activity
A = np.vstack([np.ones(N), act]).T
c1 = np.linalg.lstsq(A, p1, rcond=None)[0]
c2 = np.linalg.lstsq(A, p2, rcond=None)[0]
print(f"fit P1 = {c1[0]:.0f} + {c1[1]:.2f}*active ; P2 = {c2[0]:.0f} + {c2[1]:.2f}*active")
b.close()
