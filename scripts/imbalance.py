"""C1 load-imbalance probe: kernel time of 1024 copies of one env (heavy / median / light) vs the
real mixed batch. If copies of the heaviest env take as long as the mixed batch, the kernel time is
set by the slowest CTA (one wave of 1024 CTAs)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

N, H, W, STEPS = 1024, 128, 128, 200
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)
stream = torch.cuda.Stream()


def time_batch(fc, el, ws, wd, st, streams, reps=5):
    b = eb.Batch(N, H, W, stream=stream.cuda_stream)
    b.set_terrain(fc, el, t.class_veg, t.class_den, 30.0)
    b.set_wind(ws, wd)
    dev = torch.from_numpy(np.ascontiguousarray(st)).cuda()
    ms = []
    for i in range(reps + 2):
        with torch.cuda.stream(stream):
            eb._lib.check(eb.lib().ebl_batch_set_state_device(b.handle, dev.data_ptr()))
            b.set_key(0, 0, streams=streams)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            b.step(STEPS)
            e1.record(stream)
        e1.synchronize()
        if i >= 2:
            ms.append(e0.elapsed_time(e1))
    fin = b.get_state()
    b.close()
    return float(np.median(ms)), fin


base = np.arange(N, dtype=np.uint64)
ms, fin = time_batch(t.fuel_class, t.elevation, t.wind_speed, t.wind_direction, init, base)
burned = (fin != 0).reshape(N, -1).sum(1)
print(f"mixed batch: {ms:.3f} ms; burned cells per env: min {burned.min()} median {int(np.median(burned))} "
      f"max {burned.max()}", flush=True)
order = np.argsort(burned)
for name, e in (("heaviest", order[-1]), ("p90", order[int(0.9 * N)]), ("median", order[N // 2]),
                ("light", order[N // 10])):
    idx = np.full(N, e)
    ms1, _ = time_batch(t.fuel_class[idx], t.elevation[idx], t.wind_speed[idx], t.wind_direction[idx],
                        init[idx], np.full(N, e, dtype=np.uint64))
    print(f"{name:8s} env {e} (burned {burned[e]}): 1024 copies {ms1:.3f} ms", flush=True)
