"""Where the host-buffer (e2e) time of the C1 run goes: PCIe copies alone vs the pipelined run."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

N, H, W, STEPS = 1024, 128, 128, 200
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)
h_in = torch.from_numpy(init.copy()).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
d = torch.empty_like(h_in, device="cuda")


def tm(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


print(f"H2D 16.8 MB pinned: {tm(lambda: d.copy_(h_in, non_blocking=True)):.3f} ms")
print(f"D2H 16.8 MB pinned: {tm(lambda: h_out.copy_(d, non_blocking=True)):.3f} ms")
b = eb.Batch(N, H, W, stream=torch.cuda.current_stream().cuda_stream)
b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
b.set_wind(t.wind_speed, t.wind_direction)
L = eb.lib()


d.copy_(h_in)


def dev():
    eb._lib.check(L.ebl_batch_set_state_device(b.handle, d.data_ptr()))
    b.set_key(0, 0)
    b.step(STEPS)


print(f"device run: {tm(dev):.3f} ms")
for c in (1, 2, 4, 8, 16):
    b.set_pipeline(c)

    def run():
        b.set_key(0, 0)
        eb._lib.check(L.ebl_batch_run(b.handle, h_in.data_ptr(), STEPS, h_out.data_ptr()))
    print(f"ebl_batch_run chunks={c}: {tm(run):.3f} ms")

# Upper bound of ordering the host->device chunks by work: the same envs permuted heaviest-first
# (work proxy: cells touched by the fire at the end of the run) vs lightest-first.
b.set_pipeline(0)
b.set_key(0, 0)
eb._lib.check(L.ebl_batch_run(b.handle, h_in.data_ptr(), STEPS, h_out.data_ptr()))
work = (h_out.numpy().reshape(N, -1) != 0).sum(1)
ho = eb.host_buffer(init.shape)
print("corr(work, wind speed) %.3f" % np.corrcoef(work, t.wind_speed)[0, 1])
for name, order in (("identity", np.arange(N)), ("heaviest-first", np.argsort(-work, kind="stable")),
                    ("lightest-first", np.argsort(work, kind="stable"))):
    bp = eb.Batch(N, H, W, stream=torch.cuda.current_stream().cuda_stream)
    bp.set_terrain(t.fuel_class[order], t.elevation[order], t.class_veg, t.class_den, 30.0)
    bp.set_wind(t.wind_speed[order], t.wind_direction[order])
    hp_np = eb.host_buffer(init.shape)  # huge-page pinned: the same DMA rate for every order
    hp_np[:] = init[order]
    hp = torch.from_numpy(hp_np)
    streams = order.astype(np.uint64)
    dp = hp.cuda()

    def devp():
        eb._lib.check(L.ebl_batch_set_state_device(bp.handle, dp.data_ptr()))
        bp.set_key(0, 0, streams=streams)
        bp.step(STEPS)
    print(f"{name} device run: {tm(devp):.3f} ms")
    for c in (4, 8, 16, 32):
        bp.set_pipeline(c)

        def runp():
            bp.set_key(0, 0, streams=streams)
            eb._lib.check(L.ebl_batch_run(bp.handle, hp.data_ptr(), STEPS, ho.ctypes.data))
        print(f"{name} ebl_batch_run chunks={c}: {tm(runp):.3f} ms")
    bp.close()
