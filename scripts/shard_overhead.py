"""Halo-exchange overhead of the row-sharded landscape (C3 form) with G shards on ONE device:
fused (ebl_shards_step: peer stores from the kernels, event ordering) vs unfused (launch, then
ebl_batch_copy_rows with a host sync per copy).  All shards share the GPU, so this measures the
exchange mechanism's cost, not multi-GPU scaling.
    python scripts/shard_overhead.py [size] [steps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402
from paper_2512_06102_b200.sharded import ShardedLandscape  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
t = eb.synth_terrain(0, 1, size, size)
t.wind_speed[:] = 6.0
t.wind_direction[:] = 0.0
init = eb.synth_ignitions(0, t, 64)[0]
ref = None
for g in (1, 2, 4, 8):
    for fused in (True, False):
        sh = ShardedLandscape(t, g, fused=fused)
        ms = []
        for rep in range(3):
            sh.set_state(init)
            sh.set_key(0, 0, 0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sh.step(steps)
            sh.sync()
            ms.append(1e3 * (time.perf_counter() - t0))
        got = sh.get_state()
        if ref is None:
            ref = got
        assert np.array_equal(got, ref)
        print(f"G={g} fused={fused}: {np.median(ms):.2f} ms for {steps} steps "
              f"({size * size * steps / np.median(ms) / 1e9:.3g}e12 cell-updates/s)", flush=True)
        del sh
