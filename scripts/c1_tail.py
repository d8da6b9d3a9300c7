"""C1 critical-path probe of one library build (EBL_LIB=ab/<variant>.so, default the in-tree
build): kernel time (CUDA events on the batch stream, L2 flushed) of the mixed C1 batch and of k
copies of its heaviest / median env (k = 148: one CTA per SM; 1184: eight per SM).  Prints one
line; all variants must produce the bench's final layers (checked against the in-tree digest).
    for v in cur v1 v2; do EBL_LIB=ab/$v.so python scripts/c1_tail.py $v; done"""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06102_b200 as eb  # noqa: E402

N, H, W, STEPS = 1024, 128, 128, 200
HEAVIEST, MEDIAN = 338, 809  # C1 env ids by burned area (scripts/contention.py ranking)
name = sys.argv[1] if len(sys.argv) > 1 else os.path.basename(os.environ.get("EBL_LIB", "cur"))
t = eb.synth_terrain(0, N, H, W)
init = eb.synth_ignitions(0, t, 5)
stream = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")


def run(idx, reps=5):
    n = len(idx)
    b = eb.Batch(n, H, W, stream=stream.cuda_stream)
    b.set_terrain(t.fuel_class[idx], t.elevation[idx], t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed[idx], t.wind_direction[idx])
    dev = torch.from_numpy(np.ascontiguousarray(init[idx])).cuda()
    ms = []
    for i in range(reps + 2):
        with torch.cuda.stream(stream):
            flush.zero_()
        eb._lib.check(eb.lib().ebl_batch_set_state_device(b.handle, dev.data_ptr()))
        b.set_key(0, 0, streams=np.asarray(idx, dtype=np.uint64))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        b.step(STEPS)
        e1.record(stream)
        e1.synchronize()
        if i >= 2:
            ms.append(e0.elapsed_time(e1))
    fin = b.get_state()
    d = b.diag()
    b.close()
    return float(np.median(ms)), fin, d


ms, fin, d = run(np.arange(N))
dig = hashlib.sha1(fin.tobytes()).hexdigest()[:12]
hv = run(np.full(148, HEAVIEST))[0]
hv8 = run(np.full(1184, HEAVIEST))[0]
md = run(np.full(148, MEDIAN))[0]
print(f"{name:10s} C1 {ms:.4f} ms  heavy x148 {hv:.4f}  heavy x1184 {hv8:.4f}  median x148 {md:.4f}  "
      f"digest {dig} amb {d['ambiguous']} fb {d['fp64_fallbacks']}", flush=True)
if os.environ.get("TAIL_PROBE"):
    # the batch with its K heaviest envs (by burned area) replaced by the lightest one: the kernel
    # time the rest of the batch would take if the heavy envs ran elsewhere
    burned = (fin != 0).reshape(N, -1).sum(1)
    order = np.argsort(burned)
    row = []
    for K in (32, 64, 148, 296):
        idx = np.arange(N)
        idx[order[-K:]] = order[0]
        row.append(f"-{K}: {run(idx)[0]:.4f}")
    print(f"{name:10s} without the K heaviest: " + "  ".join(row) +
          f"   burned p50 {np.median(burned):.0f} p90 {np.percentile(burned, 90):.0f} max {burned.max()}", flush=True)
