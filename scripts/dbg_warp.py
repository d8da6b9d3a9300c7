import sys, numpy as np
sys.path.insert(0, '.')
import paper_2512_06102_b200 as eb
h = w = 64
z = np.zeros((h, w))
fire = np.zeros((h, w), np.uint8); fire[32, 32] = 1
res = {}
for k in (eb.KERNEL_RESIDENT, eb.KERNEL_WARP):
    b = eb.Batch(1, h, w)
    b.set_grid(z, z, z, z, np.zeros((h, w, 8)))
    b.set_kernel(k)
    b.set_state(fire); b.set_key(0, 0, first_stream=0)
    tr = b.step_record(6)
    res[k] = tr
for s in range(6):
    a, c = res[eb.KERNEL_RESIDENT][s, 0], res[eb.KERNEL_WARP][s, 0]
    d = np.argwhere(a != c)
    print(s, [int((a == v).sum()) for v in range(3)], [int((c == v).sum()) for v in range(3)], d[:6].tolist())
