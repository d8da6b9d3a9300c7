"""Developer tool: device deterministic forward / loss vs the fp64 oracle, step by step."""
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
for steps in (1, 2, 5, 10, 30, 100):
    b = eb.Batch(n, h, w)
    b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed, t.wind_direction)
    b.set_config(cfg)
    b.set_state(init)
    b.det_set_state_from_fire()
    b.det_forward(steps, record=True)
    un, bu, bd = b.det_get_state()
    mask = np.zeros((n, h, w))
    mask[:, 60:70, 60:70] = 1
    loss, grad = b.det_loss_grad(mask, 0.0, 1.0, 1)
    for e in range(n):
        g = O.grid_terrain(P, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                           t.wind_speed[e], t.wind_direction[e])
        u = (init[e] == 0).astype(np.float64)
        b2 = (init[e] == 1).astype(np.float64)
        d2 = (init[e] == 2).astype(np.float64)
        P.ebo_det_run(g.h, O.ptr(O.cfg_array(cfg)), steps, O.ptr(u), O.ptr(b2), O.ptr(d2))
        diff = np.abs(bu[e] - b2)
        idx = np.unravel_index(diff.argmax(), diff.shape)
        host_loss = np.mean((bu[e].astype(np.float64) + bd[e] - mask[e]) ** 2)
        ora_loss = np.mean((b2 + d2 - mask[e]) ** 2)
        lo, g6 = O._D(), np.empty(6)
        P.ebo_det_loss_grad(g.h, O.ptr(O.cfg_array(cfg)), steps, O.ptr(init[e]), O.ptr(mask[e]),
                            0.0, 1.0, 1, lo, O.ptr(g6))
        print(f"steps={steps} env={e} maxdiff_burn={diff.max():.3g} at {idx} dev={bu[e][idx]:.6g} "
              f"ora={b2[idx]:.6g} sum_burn dev={bu[e].sum():.6g} ora={b2.sum():.6g} "
              f"loss dev={loss[e]:.8g} host(dev state)={host_loss:.8g} ora_state={ora_loss:.8g} "
              f"dual={lo.value:.8g}")
        print(f"     grad dev={np.array2string(grad[e], precision=6)}\n     grad ora={np.array2string(g6, precision=6)}")
