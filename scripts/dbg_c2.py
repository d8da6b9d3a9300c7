import sys, numpy as np
sys.path.insert(0, '.')
import paper_2512_06102_b200 as eb
from oracle import oracle as O
sys.path.insert(0, 'tests')
from test_rl_gpu import _port_tanker
n, h, w, seed, steps = 16384, 64, 64, 11, int(sys.argv[1]) if len(sys.argv) > 1 else 300
t = eb.synth_terrain(seed, n, h, w)
cfg = [0.12, 0.2, 0.4, 1.0, 1.0, 0.6]
res = {}
for kernel in (eb.KERNEL_AUTO, eb.KERNEL_RESIDENT):
    env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=cfg, ignitions=5, max_steps=256)
    env.batch.set_kernel(kernel)
    env.reset(seed)
    rs, ep = env.rollout(steps)
    res[kernel] = (env.fire(), env.wet(), rs, ep, env.batch.diag())
a, b = res[eb.KERNEL_AUTO], res[eb.KERNEL_RESIDENT]
bad = np.nonzero((a[0] != b[0]).reshape(n, -1).any(1) | (a[2] != b[2]))[0]
print("differing envs:", len(bad), bad[:10], "diag", a[4], b[4])
P = O.port()
for e in bad[:3]:
    sub = eb.Terrain(t.fuel_class[[e]], t.elevation[[e]], t.wind_speed[[e]], t.wind_direction[[e]], t.class_veg, t.class_den, t.cellsize)
    want = _port_tanker(P, sub, cfg, seed, [int(e)], steps, O.TankerCfg(5, 256, 1))[0]
    print(e, "warp==port", np.array_equal(a[0][e], want["fire"]), "pooled==port", np.array_equal(b[0][e], want["fire"]),
          "rew", a[2][e], b[2][e], sum(want["rewards"]))
