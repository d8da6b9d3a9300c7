"""Pins the C restatement (oracle/ember_oracle.c) before it is trusted as the checker:
(1) against the golden fixtures produced by the reference itself (tests/golden/make_golden.py),
(2) against the reference compiled in place (oracle/_ref) on fresh inputs, bit for bit."""
import numpy as np
import pytest

from conftest import layer_cases
from oracle import oracle as O


def test_rng_kats(port, kats):
    # rng.hpp:38-58 — SURVEY §8(c) known answers + a spread of keys incl. 64-bit extremes
    for *k, want in kats["rng_word"]:
        assert hex(port.ebo_rng_word(*map(int, k))) == want
    for *k, n, want in kats["rng_below"]:
        assert port.ebo_rng_below(*map(int, k), int(n)) == int(want)
    assert port.ebo_rng_uniform(0, 0, 0, 0, 0) == 0.44705329279927764


def test_offset_angles(port):
    # grid.cpp:44-47: E=0, counter-clockwise, wrapped to [0, 2pi)
    ang = [port.ebo_offset_angle(k) for k in range(8)]
    assert ang == sorted(ang) and ang[0] == 0.0 and abs(ang[2] - np.pi / 2) < 1e-15
    assert port.ebo_wrap_angle(-0.5) == pytest.approx(2 * np.pi - 0.5, abs=1e-15)


def test_c0_kats(port, kats):
    # C0: 64x64 flat uniform, calm, ignite (32,32), SimConfig{}, RngKey{0,0,0}
    h = w = 64
    z = np.zeros((h, w))
    g = O.grid_layers(port, "port", z, z, z, z, np.zeros((h, w, 8)))
    fire = np.zeros((h, w), np.uint8)
    fire[32, 32] = 1
    for steps, want in kats["c0"].items():
        st = O.run(port, "port", g, O.DEFAULT_CFG, 0, 0, 0, int(steps), fire)
        assert [int((st == k).sum()) for k in range(3)] == want["counts"]
        assert hex(O.fnv1a64(st.tobytes())) == want["fnv1a64"]
    _, p = O.intensity(port, "port", g, O.DEFAULT_CFG, fire)
    assert p[33, 32] == kats["c0_p_one_neighbour"] == 0.11307956328284252


def test_layers_golden(port, golden_layers):
    for case in layer_cases(golden_layers):
        g = O.grid_layers(port, "port", case["speed"], case["dir"], case["veg"], case["den"],
                          case["slope8"])
        h, w = case["speed"].shape
        pot, gam = O.tables(port, "port", g, case["cfg"], h * w)
        assert np.array_equal(pot, case["pot"]) and np.array_equal(gam, case["gamma"])
        lam, p = O.intensity(port, "port", g, case["cfg"], case["probe_state"])
        assert np.array_equal(lam, case["lam"]) and np.array_equal(p, case["p"])
        traj = case["traj"]
        st = traj[0]
        for t in range(1, len(traj)):
            st = O.run(port, "port", g, case["cfg"], int(case["seed"]), t - 1, int(case["stream"]),
                       1, st)
            assert np.array_equal(st, traj[t]), f"step {t}"


def test_terrain_golden(port, golden_terrain):
    d = golden_terrain
    n = d["cls"].shape[0]
    for e in range(n):
        g = O.grid_terrain(port, "port", d["veg"][d["cls"][e]], d["den"][d["cls"][e]], d["elev"][e],
                           30.0, d["wind_speed"][e], d["wind_dir"][e])
        if e == 0:
            h, w = d["cls"].shape[1:]
            # slope_from_dem bitwise (geodata.cpp:209-229)
            assert np.array_equal(np.frombuffer(np.ctypeslib.as_array(
                (O._D * (h * w * 8)).from_address(port_slope_addr(g))), dtype=np.float64),
                d["slope0"])
        st = O.run(port, "port", g, O.DEFAULT_CFG, int(d["seed"]), 0, e, int(d["steps"]), d["init"][e])
        assert np.array_equal(st, d["final"][e])


def port_slope_addr(g):
    import ctypes as C

    class EG(C.Structure):
        _fields_ = [("h", C.c_int), ("w", C.c_int), ("speed", C.c_void_p), ("dir", C.c_void_p),
                    ("veg", C.c_void_p), ("den", C.c_void_p), ("slope8", C.c_void_p)]
    return EG.from_address(g.h).slope8


def test_rl_golden(port, golden_rl):
    ec = O.EnvCfg(20, 20, 2, 30, 0.05, 120, 1, 1, 1.0, 0.0, 0.0, 0.0,
                  (O._D * 6)(0.06, 0.1, 0.2, 0.5, 1.0, 0.9))
    for ep in range(3):
        s = O.EnvSt()
        fire = np.zeros((20, 20), np.uint8)
        port.ebo_env_reset(ec, 11, ep, s, O.ptr(fire))
        states = golden_rl[f"e{ep}_states"]
        agents = golden_rl[f"e{ep}_agents"]
        assert np.array_equal(fire, states[0])
        assert [s.agent_row, s.agent_col, s.water, s.step, s.done] == list(agents[0])
        for t, (a, rw_want) in enumerate(zip(golden_rl[f"e{ep}_actions"], golden_rl[f"e{ep}_rewards"])):
            assert port.ebo_random_policy(11, s.step, ep) == a
            s2, f2, rw = O.EnvSt(), np.empty_like(fire), O._D()
            obs = np.empty(78)
            assert port.ebo_env_step(ec, s, O.ptr(fire), int(a), s2, O.ptr(f2), rw, O.ptr(obs)) == 0
            s, fire = s2, f2
            assert rw.value == rw_want
            assert np.array_equal(fire, states[t + 1])
            assert [s.agent_row, s.agent_col, s.water, s.step, s.done] == list(agents[t + 1])
        assert np.array_equal(obs, golden_rl[f"e{ep}_last_obs"])
        # stepping a finished episode is a logic_error in the reference (rl_env.cpp:173)
        assert port.ebo_env_step(ec, s, O.ptr(fire), 0, O.EnvSt(), O.ptr(f2), O._D(), None) == -1


# ---- live comparisons against the reference compiled in place ----------------------------------
@pytest.mark.parametrize("seed,h,w,steps", [(1, 7, 7, 25), (2, 16, 48, 30), (3, 40, 3, 30)])
def test_port_vs_ref_layers(port, ref, seed, h, w, steps):
    rs = np.random.default_rng(seed)
    L = dict(speed=3.0 * rs.random((h, w)), dir=20 * rs.random((h, w)) - 10,
             veg=2.4 * rs.random((h, w)) - 1.2, den=2.4 * rs.random((h, w)) - 1.2,
             slope8=rs.random((h, w, 8)) - 0.5)
    cfg = [0.3, 0.25, 0.5, 1.5, 1.2, 0.7]
    gp = O.grid_layers(port, "port", *L.values())
    gr = O.grid_layers(ref, "ref", *L.values())
    f0 = (rs.random((h, w)) < 0.1).astype(np.uint8)
    assert np.array_equal(O.tables(port, "port", gp, cfg, h * w)[0], O.tables(ref, "ref", gr, cfg, h * w)[0])
    a = O.run(port, "port", gp, cfg, 77, 5, 3, steps, f0)
    b = O.run(ref, "ref", gr, cfg, 77, 5, 3, steps, f0)
    assert np.array_equal(a, b)


def test_port_vs_ref_terrain(port, ref):
    rs = np.random.default_rng(9)
    h, w = 48, 40
    veg = np.array([0.4, 0.25, 0.15, 0.0, -0.8, -0.7, -1.0, -1.0, -0.4, -0.2, -0.3])
    den = np.array([0.3, 0.1, -0.1, -0.2, -0.8, -0.6, -1.0, -1.0, -0.3, -0.1, -0.4])
    cls = rs.integers(0, 11, (h, w))
    el = (300 * rs.random((h, w))).astype(np.float32)
    gp = O.grid_terrain(port, "port", veg[cls], den[cls], el, 30.0, 6.0, 0.0)
    gr = O.grid_terrain(ref, "ref", veg[cls], den[cls], el, 30.0, 6.0, 0.0)
    f0 = np.zeros((h, w), np.uint8)
    f0[24, 20] = f0[10, 5] = 1
    for cfg in (O.DEFAULT_CFG, [0.5, 0.2, 0.4, 3.0, 1.0, 0.8]):
        lp, pp = O.intensity(port, "port", gp, cfg, f0)
        lr, pr = O.intensity(ref, "ref", gr, cfg, f0)
        assert np.array_equal(lp, lr) and np.array_equal(pp, pr)
        assert np.array_equal(O.run(port, "port", gp, cfg, 5, 0, 1, 50, f0),
                              O.run(ref, "ref", gr, cfg, 5, 0, 1, 50, f0))


def test_port_vs_ref_batch(port, ref):
    # step_batch lockstep (engine.cpp:134-159) == solo runs on streams first_stream+m
    h, w = 10, 10
    rs = np.random.default_rng(61)
    L = dict(speed=2 * rs.random((h, w)), dir=6.28 * rs.random((h, w)), veg=rs.random((h, w)) - 0.3,
             den=rs.random((h, w)) - 0.3, slope8=0.5 * rs.random((h, w, 8)) - 0.25)
    gr = O.grid_layers(ref, "ref", *L.values())
    gp = O.grid_layers(port, "port", *L.values())
    f0 = np.zeros((h, w), np.uint8)
    f0[5, 5] = 1
    cfg = np.array([0.22, 0.2, 0.4, 1.0, 1.0, 0.6])
    out = np.empty((8, h, w), np.uint8)
    assert ref.ref_step_batch(gr.h, O.ptr(cfg), 123, 4, 8, 15, O.ptr(f0), O.ptr(out)) == 0
    for m in range(8):
        assert np.array_equal(out[m], O.run(port, "port", gp, cfg, 123, 0, 4 + m, 15, f0))


@pytest.mark.parametrize("bce_w,mse_w,pool", [(0.0, 1.0, 1), (1.0, 1.0, 4), (0.5, 2.0, 3)])
def test_port_vs_ref_dual_loss_grad(port, ref, bce_w, mse_w, pool):
    # C4 gradient oracle: run_deterministic<Dual<6>> + loss, restated vs the reference, bitwise
    rs = np.random.default_rng(int(bce_w * 10 + pool))
    h, w = 14, 11
    veg = np.array([0.4, 0.25, 0.15, 0.0, -0.8, -0.7, -1.0, -1.0, -0.4, -0.2, -0.3])
    den = np.array([0.3, 0.1, -0.1, -0.2, -0.8, -0.6, -1.0, -1.0, -0.3, -0.1, -0.4])
    cls = rs.integers(0, 11, (h, w))
    el = (200 * rs.random((h, w))).astype(np.float32)
    gp = O.grid_terrain(port, "port", veg[cls], den[cls], el, 30.0, 4.0, 1.0)
    gr = O.grid_terrain(ref, "ref", veg[cls], den[cls], el, 30.0, 4.0, 1.0)
    f0 = np.zeros((h, w), np.uint8)
    f0[7, 5] = f0[2, 2] = 1
    mask = (rs.random((h, w)) < 0.3).astype(np.float64)
    mask[0, 0] = 1.0
    cfg = O.cfg_array([0.2, 0.15, 0.3, 1.2, 0.9, 0.65])
    out = {}
    for L, kind in ((port, "port"), (ref, "ref")):
        loss, g6 = O._D(), np.empty(6)
        fn = L.ebo_det_loss_grad if kind == "port" else L.ref_loss_grad
        (gp if kind == "port" else gr)
        rc = fn((gp if kind == "port" else gr).h, O.ptr(cfg), 20, O.ptr(f0), O.ptr(mask), bce_w, mse_w,
                pool, loss, O.ptr(g6))
        assert rc in (None, 0)
        out[kind] = (loss.value, g6)
    assert out["port"][0] == out["ref"][0]
    assert np.array_equal(out["port"][1], out["ref"][1])
    assert np.abs(out["ref"][1]).max() > 0


def _calib_case(seed=3, h=20, w=17):
    rs = np.random.default_rng(seed)
    L = dict(speed=np.full((h, w), 1.5), dir=np.full((h, w), 0.9), veg=rs.random((h, w)) * 0.6 + 0.1,
             den=rs.random((h, w)) * 0.5 + 0.1, slope8=0.4 * rs.random((h, w, 8)) - 0.2)
    fire = np.zeros((h, w), np.uint8)
    fire[h // 2, w // 2] = 1
    planes = [(fire == k).astype(np.float64) for k in (0, 1, 2)]
    return L, planes


def test_port_vs_ref_calibrate(port, ref):
    # calibrate.cpp:104-167: Adam through ThetaTransform on Dual<6> rollouts, bitwise
    L, planes = _calib_case()
    gp = O.grid_layers(port, "port", *L.values())
    gr = O.grid_layers(ref, "ref", *L.values())
    true_theta = [0.22, 0.15, 0.3, 0.8, 1.1, 0.7]
    un, bu, bd = [p.copy() for p in planes]
    port.ebo_det_run(gp.h, O.ptr(O.cfg_array(true_theta)), 12, O.ptr(un), O.ptr(bu), O.ptr(bd))
    mask = ((bu + bd) >= 0.5).astype(np.float64)
    init = [0.15, 0.2, 0.25, 1.1, 0.9, 0.6]
    for kw in (dict(), dict(bce_w=0.0, mse_w=1.0, pool=1), dict(optimize=[1, 0, 1, 1, 0, 1])):
        a = O.calibrate(port, "port", gp, planes, mask, 12, 8, init, **kw)
        b = O.calibrate(ref, "ref", gr, planes, mask, 12, 8, init, **kw)
        assert a[0] == b[0] == 0
        for x, y in zip(a[1:], b[1:]):
            assert np.array_equal(np.asarray(x), np.asarray(y))
    assert a[4] < a[1][0]  # the loss went down
    # invalid init (p_continue outside (0,1)) is rejected by both
    assert O.calibrate(port, "port", gp, planes, mask, 12, 2, [0.1, 0, 0, 0, 1, 1.5])[0] == -2
    assert O.calibrate(ref, "ref", gr, planes, mask, 12, 2, [0.1, 0, 0, 0, 1, 1.5])[0] == -1


def test_port_vs_ref_dem_nodata(port, ref):
    # slope_from_dem (geodata.cpp:209-229): NaN elevation = nodata, slope 0 from and toward it
    rs = np.random.default_rng(71)
    h, w = 13, 9
    el = (300 * rs.random((h, w))).astype(np.float32)
    el[0, 0] = el[6, 4] = el[12, 8] = el[3, 8] = np.nan
    veg, den = rs.random((h, w)) - 0.3, rs.random((h, w)) - 0.3
    gp = O.grid_terrain(port, "port", veg, den, el, 25.0, 3.0, 2.0)
    gr = O.grid_terrain(ref, "ref", veg, den, el, 25.0, 3.0, 2.0)
    cfg = np.array([0.3, 0.2, 0.4, 1.5, 1.0, 0.6])
    pp, gmp = O.tables(port, "port", gp, cfg, h * w)
    pr, gmr = O.tables(ref, "ref", gr, cfg, h * w)
    assert np.array_equal(pp, pr) and np.array_equal(gmp, gmr)
    s = np.empty(h * w * 8)
    ref.ref_grid_slope(gr.h, O.ptr(s))
    s = s.reshape(h, w, 8)
    assert (s[6, 4] == 0).all() and s[5, 4, 2] == 0.0 and s[7, 4, 6] == 0.0  # N of / S of nodata
    f0 = np.zeros((h, w), np.uint8)
    f0[6, 3] = f0[1, 1] = 1
    assert np.array_equal(O.run(port, "port", gp, cfg, 9, 0, 2, 40, f0),
                          O.run(ref, "ref", gr, cfg, 9, 0, 2, 40, f0))


def landcover_restated(lc, elev, table, fallback):
    """fuel_layers (geodata.cpp:324-345) in numpy: nodata (NaN landcover or DEM) -> (-1, -1)."""
    veg = np.full(lc.shape, -1.0)
    den = np.full(lc.shape, -1.0)
    for idx in np.ndindex(lc.shape):
        if np.isnan(lc[idx]) or np.isnan(elev[idx]):
            continue
        v, d = table.get(int(lc[idx]), fallback)
        veg[idx], den[idx] = v, d
    return veg, den


def test_ref_landcover_mapping(ref):
    rs = np.random.default_rng(72)
    h, w = 12, 10
    el = (100 * rs.random((h, w))).astype(np.float32)
    el[2, 2] = np.nan
    lc = rs.choice([10, 20, 30, 40, 50, 60, 70, 80, 90, 95, 100, 7], (h, w)).astype(np.float64)
    lc[5, 5] = np.nan
    tab = {10: (0.4, 0.3), 20: (0.25, 0.1), 30: (0.15, -0.1), 40: (0.0, -0.2), 50: (-0.8, -0.8),
           60: (-0.7, -0.6), 70: (-1.0, -1.0), 80: (-1.0, -1.0), 90: (-0.4, -0.3), 95: (-0.2, -0.1),
           100: (-0.3, -0.4)}
    with pytest.raises(RuntimeError, match="no entry for landcover code 7"):
        O.grid_from_rasters(ref, el, lc, tab)
    _, v, d = O.grid_from_rasters(ref, el, lc, tab, fallback=(0.05, -0.05))
    rv, rd = landcover_restated(lc, el, tab, (0.05, -0.05))
    assert np.array_equal(v, rv) and np.array_equal(d, rd)
    with pytest.raises(RuntimeError, match="must lie in"):
        O.grid_from_rasters(ref, el, lc, {10: (1.5, 0.0)}, fallback=(0, 0))


@pytest.mark.parametrize("n,h,w,env0", [(8, 128, 128, 0), (3, 64, 64, 1024), (2, 130, 520, 5),
                                        (2, 2, 2, 0), (2, 7, 300, 3), (2, 256, 256, 7000)])
def test_synth_inputs_port_equals_product_generator(n, h, w, env0):
    """The port's restatement of the benchmark input generator (used by bench.py's CPU arms so
    they never load the product library) is bit-identical to ebl_synth_terrain/_ignitions."""
    import paper_2512_06102_b200 as eb
    a = O.SynthTerrain(0, n, h, w, env_id0=env0)
    b = eb.synth_terrain(0, n, h, w, env_id0=env0)
    assert np.array_equal(a.fuel_class, b.fuel_class)
    assert np.array_equal(a.elevation.view(np.uint32), b.elevation.view(np.uint32))
    assert np.array_equal(a.wind_speed, b.wind_speed)
    assert np.array_equal(a.wind_direction, b.wind_direction)
    assert np.array_equal(a.class_veg, b.class_veg) and np.array_equal(a.class_den, b.class_den)
    for k in (1, 5, 64):
        assert np.array_equal(a.ignitions(k), eb.synth_ignitions(0, b, k, env_id0=env0))
