"""Developer tool: locate the first step/cell where the device path and the oracle diverge
on C1-shaped inputs, and print the draw vs threshold there.  Usage:
    python scripts/debug_parity.py [n_envs] [steps]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2512_06102_b200 as eb  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
P = O.port()
t = eb.synth_terrain(0, n, 128, 128)
init = eb.synth_ignitions(0, t, 5)
for cfg in ([0.12, 0.2, 0.4, 1.0, 1.0, 0.6], [0.3, 0.1, 0.3, 2.0, 1.5, 0.8],
            [0.12, 0.2, 0.4, 1.0, 1.0, 0.95]):
    for kernel in (eb.KERNEL_TILED, eb.KERNEL_RESIDENT):
        b = eb.Batch(n, 128, 128)
        b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
        b.set_wind(t.wind_speed, t.wind_direction)
        b.set_config(cfg)
        b.set_kernel(kernel)
        b.set_state(init)
        b.set_key(0, 0)
        grids = [O.grid_terrain(P, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                                t.wind_speed[e], t.wind_direction[e]) for e in range(n)]
        cur = init.copy()
        bad = False
        for s in range(steps):
            b.step(1)
            got = b.get_state()
            for e in range(n):
                want = O.run(P, "port", grids[e], cfg, 0, s, e, 1, cur[e])
                if not np.array_equal(got[e], want):
                    cells = np.argwhere(got[e] != want)
                    print(f"cfg={cfg} kernel={kernel} env={e} step={s} cells={cells[:4].tolist()} "
                          f"got={got[e][tuple(cells[0])]} want={want[tuple(cells[0])]} "
                          f"prev={cur[e][tuple(cells[0])]}")
                    lam, p = O.intensity(P, "port", grids[e], cfg, cur[e])
                    r, c = cells[0]
                    u = P.ebo_rng_uniform(0, s, e, int(r * 128 + c), 0)
                    b2 = eb.Batch(1, 128, 128)
                    b2.set_terrain(t.fuel_class[e:e + 1], t.elevation[e:e + 1], t.class_veg,
                                   t.class_den, 30.0)
                    b2.set_wind(t.wind_speed[e:e + 1], t.wind_direction[e:e + 1])
                    b2.set_config(cfg)
                    b2.set_state(cur[e])
                    l32, p32 = b2.intensity()
                    print(f"   u={u!r} p64={p[r, c]!r} lam64={lam[r, c]!r} p32={p32[0, r, c]!r} "
                          f"lam32={l32[0, r, c]!r} rel={(p32[0, r, c] - p[r, c]) / p[r, c]:.3g}")
                    bad = True
                    break
            if bad:
                break
            cur = got
        print(f"cfg={cfg} kernel={kernel}: {'DIVERGED' if bad else 'ok'} diag={b.diag()}", flush=True)
