"""Phase profile of the warp-local kernel (EBL_PHASE_PROF build: EBL_LIB=ab/prof.so): per env
cycles/step of the slowest warp's dense pass and decide passes, passes per step, barrier wait;
k copies of the heaviest / median / light C1 env, one CTA per SM and 8 per SM."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

VARIANT = sys.argv[1] if len(sys.argv) > 1 else ""

N, H, W, STEPS = 1024, 128, 128, 200
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)
for name, e in (("heaviest", 338), ("median", 809), ("light", 760)):
    for k in (148, 1184):
        idx = np.full(k, e)
        b = eb.Batch(k, H, W)
        b.set_terrain(t.fuel_class[idx], t.elevation[idx], t.class_veg, t.class_den, 30.0)
        b.set_wind(t.wind_speed[idx], t.wind_direction[idx])
        b.set_kernel(6)
        eb._lib.check(eb.lib().ebl_batch_set_profiling(b.handle, 1))
        for _ in range(2):
            b.set_state(init[idx])
            b.set_key(0, 0, streams=idx.astype(np.uint64))
            b.step(STEPS)
        pr = np.zeros((k, 10), np.int64)
        eb._lib.check(eb.lib().ebl_batch_profile(b.handle, pr.ctypes.data))
        p = pr.mean(0) / STEPS
        print(f"{VARIANT} {name:8s} x{k:4d}: step {p[6]:6.0f}  dense(max warp) {p[0]:5.0f}  decide(max warp) {p[1]:6.0f}  "
              f"barrier wait(max) {p[7]:5.0f}  passes/step: max-warp {p[4]:4.2f} all {p[5]:4.2f}  "
              f"locate {p[8]:5.0f} body(lane 0, candidates) {p[9]:5.0f} load latency(lane 0) {p[3]:5.0f}", flush=True)
        b.close()
