import sys, numpy as np
sys.path.insert(0, '.')
import paper_2512_06102_b200 as eb
h, w = int(sys.argv[1]), int(sys.argv[2])
rs = np.random.default_rng(h * 1000 + w)
n = 5
cls = rs.integers(0, 11, (n, h, w)).astype(np.uint8)
el = (400 * rs.random((n, h, w))).astype(np.float32)
_, veg, den = eb.worldcover_palette()
init = (rs.random((n, h, w)) < 0.15).astype(np.uint8)
init[rs.random((n, h, w)) < 0.1] = 2
init[rs.random((n, h, w)) < 0.01] = 7
variants = [(eb.KERNEL_TILED, None), (eb.KERNEL_AUTO, None), (eb.KERNEL_BLOCKED, None),
            (eb.KERNEL_AUTO, (8, 32, 3)), (eb.KERNEL_AUTO, (5, 64, 1)), (eb.KERNEL_AUTO, (16, 96, 7)), (eb.KERNEL_PAIRED, None)]
for kernel, tiling in variants:
    try:
        b = eb.Batch(n, h, w)
        b.set_terrain(cls, el, veg, den, 25.0)
        b.set_wind(rs.random(n) * 0 + 7.0, [0.3, 1.0, 2.0, 4.0, 6.0])
        b.set_config([0.4, 0.2, 0.4, 1.0, 1.0, 0.7])
        b.set_kernel(kernel)
        if tiling:
            b.set_tiling(*tiling)
        b.set_state(init)
        b.set_key(9, 3, first_stream=100)
        b.step(25)
        st = b.get_state()
        print("ok", kernel, tiling, flush=True)
    except Exception as e:
        print("FAIL", kernel, tiling, e, flush=True)
        break
