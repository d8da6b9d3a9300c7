"""RL step on device vs the reference (golden episodes) and the C oracle (batched, tanker)."""
import numpy as np
import pytest

import paper_2512_06102_b200 as eb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _agents(env):
    return [[s.agent_row, s.agent_col, s.water, s.step, s.done] for s in env.env_states()]


def test_reference_env_golden_episodes(golden_rl):
    # FireSuppressionEnv default_preset, random_policy episodes keyed (11, step, stream=ep)
    env = eb.VecFireEnv(3)
    env.reset(11, streams=[0, 1, 2])
    fires = env.fire()
    ag = _agents(env)
    for ep in range(3):
        assert np.array_equal(fires[ep], golden_rl[f"e{ep}_states"][0])
        assert ag[ep] == list(golden_rl[f"e{ep}_agents"][0])
    # host-supplied actions (the golden ones), envs finish at different times: step one env at a time
    for ep in range(3):
        acts = golden_rl[f"e{ep}_actions"]
        e1 = eb.VecFireEnv(1)
        e1.reset(11, streams=[ep])
        for t, a in enumerate(acts):
            r, d = e1.step([int(a)])
            assert r[0] == golden_rl[f"e{ep}_rewards"][t]
            assert np.array_equal(e1.fire()[0], golden_rl[f"e{ep}_states"][t + 1])
            assert _agents(e1)[0] == list(golden_rl[f"e{ep}_agents"][t + 1])
            assert bool(d[0]) == bool(golden_rl[f"e{ep}_agents"][t + 1][4])
        assert np.array_equal(e1.observe()[0], golden_rl[f"e{ep}_last_obs"])
        with pytest.raises(eb.LogicError):
            e1.step([0])  # rl_env.cpp:173
        with pytest.raises(eb.OutOfRange):
            e1.step([10])


def test_reference_env_device_policy_matches_golden(golden_rl):
    # actions=None -> device random_policy (rl_env.cpp:237-239); one env per episode length
    for ep in range(3):
        e1 = eb.VecFireEnv(1)
        e1.reset(11, streams=[ep])
        for t in range(len(golden_rl[f"e{ep}_actions"])):
            r, _ = e1.step(None)
            assert r[0] == golden_rl[f"e{ep}_rewards"][t]
        assert np.array_equal(e1.fire()[0], golden_rl[f"e{ep}_states"][-1])


def test_reference_env_batch_vs_port(port):
    cfg = eb.default_preset()
    cfg.ignition_count = 4
    cfg.waste_water = 0
    n = 64
    env = eb.VecFireEnv(n, cfg)
    env.reset(5)
    ec = O.EnvCfg(cfg.height, cfg.width, cfg.window_radius, cfg.water_capacity, cfg.burn_penalty,
                  cfg.max_episode_steps, cfg.ignition_count, cfg.waste_water, cfg.wind_speed,
                  cfg.wind_direction, cfg.fuel_veg, cfg.fuel_den, (O._D * 6)(*cfg.spread.as_list()))
    states, fires = [], []
    for e in range(n):
        s = O.EnvSt()
        f = np.zeros((cfg.height, cfg.width), np.uint8)
        port.ebo_env_reset(ec, 5, e, s, O.ptr(f))
        states.append(s)
        fires.append(f)
    assert np.array_equal(env.fire(), np.stack(fires))
    rs = np.random.default_rng(0)
    for t in range(40):
        live = [e for e in range(n) if not states[e].done]
        if not live:
            break
        acts = rs.integers(0, 10, n).astype(np.int32)
        # finished envs must not be stepped (logic_error): give them their own batch view
        sub = eb.VecFireEnv(len(live), cfg)
        sub.reset(5, streams=live)
        sub.set_fire(np.stack([fires[e] for e in live]))
        sub.set_env_states([eb.EnvState(states[e].agent_row, states[e].agent_col, states[e].water,
                                        states[e].step, 5, e, states[e].done, 0) for e in live])
        r, d = sub.step(acts[live])
        obs = sub.observe()
        for i, e in enumerate(live):
            s2, f2, rw = O.EnvSt(), np.empty_like(fires[e]), O._D()
            ob = np.empty(78)
            assert port.ebo_env_step(ec, states[e], O.ptr(fires[e]), int(acts[e]), s2, O.ptr(f2), rw,
                                     O.ptr(ob)) == 0
            states[e], fires[e] = s2, f2
            assert r[i] == rw.value and bool(d[i]) == bool(s2.done)
            assert np.array_equal(sub.fire()[i], f2)
            assert np.array_equal(obs[i], ob)


def _port_tanker(port, t: eb.Terrain, cfg, seed, env_ids, n_steps, tc, actions=None):
    n, h, w = t.fuel_class.shape
    out = []
    for i, e in enumerate(env_ids):
        g = O.grid_terrain(port, "port", t.veg()[i], t.den()[i], t.elevation[i], t.cellsize,
                           t.wind_speed[i], t.wind_direction[i])
        pot, gam = O.tables(port, "port", g, cfg, h * w)
        s = O.TankerSt()
        fire = np.zeros((h, w), np.uint8)
        wet = np.zeros((h, w), np.uint8)
        port.ebo_tanker_reset(g.h, tc, seed, e, 0, s, O.ptr(fire), O.ptr(wet))
        rewards, dones = [], []
        for k in range(n_steps):
            a = (port.ebo_tanker_policy(seed, e, s, h * w) if actions is None else int(actions[k][i]))
            rw = np.zeros(1, np.float32)
            dn = np.zeros(1, np.uint8)
            port.ebo_tanker_step(g.h, O.ptr(pot), O.ptr(gam), float(cfg[5]), tc, seed, e, a, s,
                                 O.ptr(fire), O.ptr(wet), O.ptr(rw), O.ptr(dn))
            rewards.append(float(rw[0]))
            dones.append(int(dn[0]))
        out.append(dict(fire=fire, wet=wet, rewards=rewards, dones=dones, step=s.step,
                        episode=s.episode))
    return out


# warp-local bit-plane (AUTO) / pooled-list bit-plane (RESIDENT) / byte kernel (TILED)
@pytest.mark.parametrize("kernel", [eb.KERNEL_AUTO, eb.KERNEL_RESIDENT, eb.KERNEL_TILED])
@pytest.mark.parametrize("fused", [False, True])
def test_tanker_vs_port(port, fused, kernel):
    n, h, w, seed, steps = 24, 64, 64, 7, 300
    t = eb.synth_terrain(seed, n, h, w)
    cfg = [0.12, 0.2, 0.4, 1.0, 1.0, 0.6]
    env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=cfg, ignitions=5, max_steps=256)
    env.batch.set_kernel(kernel)
    env.reset(seed)
    tc = O.TankerCfg(5, 256, 1)
    want = _port_tanker(port, t, cfg, seed, list(range(n)), steps, tc)
    if fused:
        rs, ep = env.rollout(steps)
        for e in range(n):
            assert rs[e] == sum(want[e]["rewards"])
            assert ep[e] == sum(want[e]["dones"])
    else:
        for k in range(steps):
            r, d = env.step(None)
            for e in range(n):
                assert r[e] == want[e]["rewards"][k], (e, k)
                assert d[e] == want[e]["dones"][k], (e, k)
    fire, wet = env.fire(), env.wet()
    st = env.env_states()
    for e in range(n):
        assert np.array_equal(fire[e], want[e]["fire"])
        assert np.array_equal(wet[e], want[e]["wet"])
        assert st[e].step == want[e]["step"] and st[e].episode == want[e]["episode"]
    assert sum(sum(x["dones"]) for x in want) > 0, "test should cover auto-reset"


@pytest.mark.parametrize("kernel,h,w", [(eb.KERNEL_AUTO, 32, 48), (eb.KERNEL_TILED, 32, 48),
                                          (eb.KERNEL_AUTO, 17, 45), (eb.KERNEL_RESIDENT, 17, 45),
                                          (eb.KERNEL_AUTO, 140, 33)])
def test_tanker_host_actions(port, kernel, h, w):
    n, seed, steps = 8, 3, 40
    t = eb.synth_terrain(seed, n, h, w)
    env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=None, ignitions=3, max_steps=256)
    env.batch.set_kernel(kernel)
    env.reset(seed)
    rs = np.random.default_rng(1)
    acts = rs.integers(0, h * w, (steps, n)).astype(np.int32)
    want = _port_tanker(port, t, O.DEFAULT_CFG, seed, list(range(n)), steps, O.TankerCfg(3, 256, 1),
                        actions=acts)
    for k in range(steps):
        r, _ = env.step(acts[k])
        assert [want[e]["rewards"][k] for e in range(n)] == r.tolist()
    assert np.array_equal(env.fire(), np.stack([x["fire"] for x in want]))


def test_tanker_bit_resident_state_sync():
    """The warp-local tanker keeps its layers bit-resident between ebl_rl_step calls: every other
    entry point (state read/write, wet read, observe-free reset with a mask) must see and overwrite
    the current layers.  Interleaved with those calls, AUTO matches the byte-layer RESIDENT kernel
    step for step, including a host edit of the fire layer mid-run."""
    n, h, w, seed = 16, 64, 64, 5
    t = eb.synth_terrain(seed, n, h, w)
    runs = {}
    for kernel in (eb.KERNEL_AUTO, eb.KERNEL_RESIDENT):
        env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=None, ignitions=4, max_steps=256)
        env.batch.set_kernel(kernel)
        env.reset(seed)
        log = []
        for k in range(60):
            r, d = env.step(None)
            log.append((r.copy(), d.copy()))
            if k % 7 == 3:
                log.append((env.fire(), env.wet()))
            if k == 20:  # host edit: ignite a burnable-agnostic corner cell in every env
                f = env.fire()
                f[:, 0, 0] = np.where(f[:, 0, 0] == 0, 1, f[:, 0, 0])
                env.set_fire(f)
            if k == 40:
                mask = np.zeros(n, np.uint8)
                mask[::3] = 1
                env.reset(seed + 1, mask=mask)
        log.append((env.fire(), env.wet()))
        runs[kernel] = log
    for x, y in zip(runs[eb.KERNEL_AUTO], runs[eb.KERNEL_RESIDENT]):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])


@pytest.mark.slow
def test_c2_full_size_rollout(port):
    """BASELINE C2 at full size (16384 envs of 64 x 64, device random (x, y) policy, 256-step cap,
    auto-reset): the warp-local and the pooled-list tanker kernels agree bit for bit over a 300-step
    fused rollout (layers, wet layers, episode counters, reward sums), and envs sampled across the
    batch (every 16th: 1024 envs) match the C restatement's layers, wet layers, reward sums and
    episode counts."""
    n, h, w, seed, steps = 16384, 64, 64, 11, 300
    t = eb.synth_terrain(seed, n, h, w)
    cfg = [0.12, 0.2, 0.4, 1.0, 1.0, 0.6]
    res = {}
    for kernel in (eb.KERNEL_AUTO, eb.KERNEL_RESIDENT):
        env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=cfg, ignitions=5, max_steps=256)
        env.batch.set_kernel(kernel)
        env.reset(seed)
        rs, ep = env.rollout(steps)
        st = env.env_states()
        res[kernel] = (env.fire(), env.wet(), rs, ep, [(s.step, s.episode) for s in st])
    a, b = res[eb.KERNEL_AUTO], res[eb.KERNEL_RESIDENT]
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(x, y)
    assert a[4] == b[4]
    assert a[3].sum() > n // 2, "most envs should finish an episode within 300 steps"
    # every 16th env of the batch (1024 envs, all across it) vs the C restatement, OpenMP over envs
    ids = np.arange(0, n, 16)
    want = O.tanker_run_envs(t, ids, cfg, seed, steps)
    assert np.array_equal(a[0][ids], want["fire"]) and np.array_equal(a[1][ids], want["wet"])
    assert np.array_equal(a[2][ids], want["reward"]) and np.array_equal(a[3][ids], want["episodes"])


def test_tanker_learner_in_the_loop_device_io(port):
    """A learner in the loop on the device (north_star (4): no host round trip): each step the
    policy reads the device observation (ebl_rl_observe_device: FireState | wet << 2), picks the
    first burning cell of every env with torch ops on the GPU, and ebl_rl_step(device_io=1) takes
    those device actions and writes reward/done to device tensors.  Rewards, dones, the final
    layers and the observation equal the C restatement driven by the same actions."""
    import torch
    n, h, w, seed, steps = 12, 64, 64, 9, 80
    t = eb.synth_terrain(seed, n, h, w)
    env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=None, ignitions=5, max_steps=256)
    env.reset(seed)
    dev = "cuda:0"
    obs = torch.empty((n, h, w), dtype=torch.uint8, device=dev)
    rew = torch.empty(n, dtype=torch.float64, device=dev)
    done = torch.empty(n, dtype=torch.uint8, device=dev)
    acts, rews, dones = [], [], []
    cur = torch.cuda.current_stream()
    for k in range(steps):
        env.observe_device(obs)
        env.batch.sync()  # the batch stream -> torch's stream (the policy reads obs)
        burning = (obs & 3).view(n, -1) == 1
        a = torch.where(burning.any(1), burning.to(torch.int8).argmax(1), torch.full((n,), 17, device=dev))
        a = a.to(torch.int32).contiguous()
        cur.synchronize()
        env.step_device(a, rew, done)
        env.batch.sync()
        acts.append(a.cpu().numpy())
        rews.append(rew.cpu().numpy().copy())
        dones.append(done.cpu().numpy().copy())
    want = _port_tanker(port, t, O.DEFAULT_CFG, seed, list(range(n)), steps, O.TankerCfg(5, 256, 1),
                        actions=np.stack(acts))
    for e in range(n):
        assert [r[e] for r in rews] == want[e]["rewards"], e
        assert [int(d[e]) for d in dones] == want[e]["dones"], e
    env.observe_device(obs)
    env.batch.sync()
    fire = np.stack([x["fire"] for x in want])
    wet = np.stack([x["wet"] for x in want])
    assert np.array_equal(obs.cpu().numpy(), fire | (wet << 2))
    assert np.array_equal(env.fire(), fire) and np.array_equal(env.wet(), wet)


def test_tanker_host_step_mapped_buffers(port):
    """ebl_rl_step with host buffers in mapped pinned memory (eb.host_buffer): the kernel writes
    reward / done straight through the mapping (no copy after the step) and the call returns them
    complete -- rewards, dones and the final layers equal the C restatement driven by the same
    actions, and equal the same steps with pageable buffers (DMA copies)."""
    n, h, w, seed, steps = 16, 64, 64, 4, 70
    t = eb.synth_terrain(seed, n, h, w)
    rs = np.random.default_rng(3)
    acts = rs.integers(0, h * w, (steps, n)).astype(np.int32)
    L = eb.lib()
    got = {}
    for mapped in (True, False):
        env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=None, ignitions=5, max_steps=256)
        env.reset(seed)
        mk = eb.host_buffer if mapped else (lambda shape, dtype=np.uint8: np.empty(shape, dtype))
        a, r, d = mk((n,), np.int32), mk((n,), np.float64), mk((n,), np.uint8)
        log = []
        for k in range(steps):
            a[:] = acts[k]
            eb._lib.check(L.ebl_rl_step(env.batch.handle, a.ctypes.data, r.ctypes.data, d.ctypes.data, 0))
            log.append((r.copy(), d.copy()))
        got[mapped] = (log, env.fire(), env.wet())
    want = _port_tanker(port, t, O.DEFAULT_CFG, seed, list(range(n)), steps, O.TankerCfg(5, 256, 1), actions=acts)
    log, fire, wet = got[True]
    for e in range(n):
        assert [x[0][e] for x in log] == want[e]["rewards"], e
        assert [int(x[1][e]) for x in log] == want[e]["dones"], e
    assert np.array_equal(fire, np.stack([x["fire"] for x in want]))
    assert np.array_equal(wet, np.stack([x["wet"] for x in want]))
    for (r1, d1), (r0, d0) in zip(got[True][0], got[False][0]):
        assert np.array_equal(r1, r0) and np.array_equal(d1, d0)
