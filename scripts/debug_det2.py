"""Developer tool: first step where the device deterministic forward departs from fp64."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2512_06102_b200 as eb  # noqa: E402
from oracle import oracle as O  # noqa: E402

P = O.port()
n, h, w, seed = 2, 128, 128, 4
t = eb.synth_terrain(seed, n, h, w)
init = eb.synth_ignitions(seed, t, 5)
cfg = [0.12, 0.2, 0.4, 1.0, 1.0, 0.6]
e = 0
g = O.grid_terrain(P, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0, t.wind_speed[e], t.wind_direction[e])
b = eb.Batch(n, h, w)
b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
b.set_wind(t.wind_speed, t.wind_direction)
b.set_config(cfg)
b.set_state(init)
b.det_set_state_from_fire()
u = (init[e] == 0).astype(np.float64)
b2 = (init[e] == 1).astype(np.float64)
d2 = (init[e] == 2).astype(np.float64)
prev = None
for s in range(1, 101):
    b.det_forward(1, record=False)
    un, bu, bd = b.det_get_state()
    pu, pb, pd = u.copy(), b2.copy(), d2.copy()
    P.ebo_det_run(g.h, O.ptr(O.cfg_array(cfg)), 1, O.ptr(u), O.ptr(b2), O.ptr(d2))
    diff = np.abs(bu[e] - b2)
    if diff.max() > 1e-4:
        r, c = np.unravel_index(diff.argmax(), diff.shape)
        print(f"step {s}: maxdiff {diff.max():.3g} at ({r},{c}) class={t.fuel_class[e, r, c]}")
        sl = (slice(max(0, r - 1), r + 2), slice(max(0, c - 1), c + 2))
        print("dev burn\n", bu[e][sl], "\nora burn\n", b2[sl], "\nprev dev burn\n", prev[1][sl],
              "\nprev ora burn\n", pb[sl], "\nprev dev un\n", prev[0][sl], "\nprev ora un\n", pu[sl])
        print("classes\n", t.fuel_class[e][sl], "\nelev\n", t.elevation[e][sl])
        break
    m = b2 > 1e-12
    rel = np.where(m, np.abs(bu[e] - b2) / np.maximum(b2, 1e-300), 0)
    rr, cc = np.unravel_index(rel.argmax(), rel.shape)
    print(f"step {s}: max rel burn err {rel.max():.3g} at ({rr},{cc}) dev={bu[e][rr, cc]:.4g} ora={b2[rr, cc]:.4g} "
          f"front cells(dev>0)={int((bu[e] > 0).sum())} (ora>0)={int((b2 > 0).sum())} "
          f"min dev un {un[e].min():.4g} min dev burn {bu[e].min():.4g}")
    if s % 5 == 0:
        print(f"step {s}: maxdiff burn {diff.max():.3g} un {np.abs(un[e] - u).max():.3g} "
              f"simplex dev {np.abs(un[e].astype(np.float64) + bu[e] + bd[e] - 1).max():.3g}")
    if len(sys.argv) > 1:  # resync the device to the oracle state: one step's error at a time
        sync = [np.array(x, dtype=np.float32) for x in (un, bu, bd)]
        sync[0][e], sync[1][e], sync[2][e] = u, b2, d2
        b.det_set_state(*sync)
    prev = (un[e].copy(), bu[e].copy(), bd[e].copy())
else:
    print("no divergence > 1e-4 per step")
