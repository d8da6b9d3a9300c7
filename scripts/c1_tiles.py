"""C1 (1024 x 128^2 x 200) as halo tiles on work lists (ebl_batch_set_tiling: tile_h x 128, 8-row
halos, 25 launches of 8 steps, quiet tiles skipped) vs the whole-env launch: kernel time (CUDA
events on the batch stream, L2 flushed) and bitwise equality.   python scripts/c1_tiles.py"""
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
dev = torch.from_numpy(init).cuda()
b = eb.Batch(N, H, W, stream=stream.cuda_stream)
b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
b.set_wind(t.wind_speed, t.wind_direction)
L = eb.lib()
ref = None
for th in [0] + [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["32", "16", "64"])]:
    b.set_tiling(th, 128, 8) if th else b.set_tiling(0)
    ms = []
    for rep in range(6):
        eb._lib.check(L.ebl_batch_set_state_device(b.handle, dev.data_ptr()))
        b.set_key(0, 0, first_stream=0)
        b.diag(reset=True)
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        b.step(STEPS)
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    d = b.diag()
    out = b.get_state()
    if ref is None:
        ref = out
    frac = d["tiles_processed"] / max(1, d["tiles_launched"])
    print(f"tile_h={th or 'whole env'}: {np.median(ms[1:]):.4f} ms  launches {d['launches']}  "
          f"tiles stepped {frac:.3f}  equal={np.array_equal(out, ref)}", flush=True)
