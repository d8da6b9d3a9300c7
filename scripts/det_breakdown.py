"""C4 time breakdown: host-timed det_set_state_from_fire / det_forward / det_loss_grad."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

n, h, w, steps = 256, 128, 128, 100
b = eb.Batch(n, h, w)
b.synth_terrain(4)
b.synth_ignitions(4, 5)
mask = (np.random.default_rng(0).random((n, h, w)) < 0.2).astype(np.float64)
b.det_set_state_from_fire()
b.det_forward(1, record=True)
for it in range(4):
    b.sync()
    t0 = time.perf_counter()
    b.det_set_state_from_fire()
    b.sync()
    t1 = time.perf_counter()
    b.det_forward(steps, record=True)
    t2 = time.perf_counter()
    b.det_loss_grad(mask, 0.0, 1.0, 1)
    t3 = time.perf_counter()
    print(f"iter {it}: from_fire {1e3*(t1-t0):.2f} ms  forward {1e3*(t2-t1):.2f} ms  loss+grad {1e3*(t3-t2):.2f} ms",
          flush=True)
