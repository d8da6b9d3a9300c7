"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.

Bar (north_star): cell states bit-exact; arrival intensity and ignition probability of the
fp32 path within 1e-5 relative; any flip must come from a draw inside the fp64 ambiguity band
(reported by the device as diag['ambiguous'], asserted 0 here)."""
import numpy as np
import pytest

import paper_2512_06102_b200 as eb
from conftest import layer_cases
from oracle import oracle as O

pytestmark = pytest.mark.gpu

KERNELS = [eb.KERNEL_TILED, eb.KERNEL_RESIDENT, eb.KERNEL_BLOCKED, eb.KERNEL_WARP]
REL_TOL = 1e-5  # north_star: lambda and p within 1e-5 relative in fp32


def _layers_batch(case, n_envs=1, kernel=eb.KERNEL_AUTO):
    h, w = case["speed"].shape
    b = eb.Batch(n_envs, h, w)
    b.set_config(list(case["cfg"]))
    b.set_grid(case["speed"], case["dir"], case["veg"], case["den"], case["slope8"])
    b.set_kernel(kernel)
    return b


def test_device_rng_kats(kats):
    keys = np.array([[int(x) for x in k[:5]] for k in kats["rng_word"]], dtype=np.uint64)
    out = np.zeros(len(keys), np.uint64)
    eb._lib.check(eb.lib().ebl_device_rng_words(len(keys), keys.ctypes.data, out.ctypes.data))
    assert [hex(int(x)) for x in out] == [k[5] for k in kats["rng_word"]]


def test_device_rng_random_keys(port):
    rs = np.random.default_rng(0)
    keys = rs.integers(0, 2**63, size=(4096, 5), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    out = np.zeros(len(keys), np.uint64)
    eb._lib.check(eb.lib().ebl_device_rng_words(len(keys), keys.ctypes.data, out.ctypes.data))
    want = [port.ebo_rng_word(*map(int, k)) for k in keys]
    assert [int(x) for x in out] == want


@pytest.mark.parametrize("kernel", KERNELS)
def test_c0_kats(kats, kernel):
    h = w = 64
    z = np.zeros((h, w))
    b = eb.Batch(1, h, w)
    b.set_grid(z, z, z, z, np.zeros((h, w, 8)))
    b.set_kernel(kernel)
    fire = np.zeros((h, w), np.uint8)
    fire[32, 32] = 1
    for steps, want in sorted(kats["c0"].items(), key=lambda kv: int(kv[0])):
        b.set_state(fire)
        b.set_key(0, 0, first_stream=0)
        b.step(int(steps))
        st = b.get_state()[0]
        assert [int((st == k).sum()) for k in range(3)] == want["counts"]
        assert hex(O.fnv1a64(st.tobytes())) == want["fnv1a64"]
        assert b.counts()[0, :3].tolist() == want["counts"]
    assert b.diag()["ambiguous"] == 0


def test_one_shot_signatures_golden(golden_layers):
    for case in layer_cases(golden_layers):
        traj = case["traj"]
        grid = dict(speed=case["speed"], dir=case["dir"], veg=case["veg"], den=case["den"],
                    slope8=case["slope8"])
        st = traj[0]
        for t in range(1, len(traj)):
            st = eb.step_stochastic(st, grid, list(case["cfg"]),
                                    (int(case["seed"]), t - 1, int(case["stream"])))
            assert np.array_equal(st, traj[t]), f"step {t}"
        fin = eb.run_stochastic(traj[0], grid, list(case["cfg"]),
                                (int(case["seed"]), 0, int(case["stream"])), len(traj) - 1)
        assert np.array_equal(fin, traj[-1])


@pytest.mark.parametrize("kernel", KERNELS)
def test_layers_golden_batch(golden_layers, kernel):
    for case in layer_cases(golden_layers):
        traj = case["traj"]
        b = _layers_batch(case, 3, kernel)
        b.set_state(traj[0])
        b.set_key(int(case["seed"]), 0, streams=[int(case["stream"])] * 3)
        for t in range(1, len(traj)):
            b.step(1)
            assert (b.get_state() == traj[t]).all(), f"step {t}"
        lam, p = b.intensity()
        b.set_state(case["probe_state"])
        lam, p = b.intensity()
        # tables form computes lambda/p in fp64 (rounded to float for the probe)
        np.testing.assert_allclose(lam[0], case["lam"], rtol=REL_TOL, atol=1e-30)
        np.testing.assert_allclose(p[0], case["p"], rtol=REL_TOL, atol=1e-30)
        assert b.diag()["ambiguous"] == 0


@pytest.mark.parametrize("kernel", KERNELS)
def test_terrain_golden(golden_terrain, kernel):
    d = golden_terrain
    n, h, w = d["cls"].shape
    b = eb.Batch(n, h, w)
    b.set_terrain(d["cls"], d["elev"], d["veg"], d["den"], 30.0)
    b.set_wind(d["wind_speed"], d["wind_dir"])
    b.set_kernel(kernel)
    b.set_state(d["init"])
    b.set_key(int(d["seed"]), 0, first_stream=0)
    b.step(int(d["steps"]))
    assert np.array_equal(b.get_state(), d["final"])
    assert b.diag()["ambiguous"] == 0


def _terrain_batch(t: eb.Terrain, cfg=None, kernel=eb.KERNEL_AUTO):
    n, h, w = t.fuel_class.shape
    b = eb.Batch(n, h, w)
    b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, t.cellsize)
    b.set_wind(t.wind_speed, t.wind_direction)
    b.set_config(cfg)
    b.set_kernel(kernel)
    return b


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("cfg", [None, [0.3, 0.1, 0.3, 2.0, 1.5, 0.8], [0.12, 0.2, 0.4, 1.0, 1.0, 0.95]])
def test_c1_shape_vs_oracle(port, kernel, cfg):
    """C1 generator at full env size (128x128, 5 ignitions, 200 steps), 12 envs vs the port."""
    n, h, w, steps, seed = 12, 128, 128, 200, 0
    t = eb.synth_terrain(seed, n, h, w)
    init = eb.synth_ignitions(seed, t, 5)
    b = _terrain_batch(t, cfg, kernel)
    b.set_state(init)
    b.set_key(seed, 0, first_stream=0)
    b.step(steps)
    got = b.get_state()
    c = O.DEFAULT_CFG if cfg is None else cfg
    for e in range(n):
        g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                           t.wind_speed[e], t.wind_direction[e])
        want = O.run(port, "port", g, c, seed, 0, e, steps, init[e])
        assert np.array_equal(got[e], want), f"env {e}: {np.argwhere(got[e] != want)[:5]}"
    cnt = b.counts()
    assert (cnt[:, :3].sum(1) == h * w).all()
    assert np.array_equal(cnt[:, 1], (got == 1).reshape(n, -1).sum(1))
    d = b.diag()
    assert d["ambiguous"] == 0


def test_intensity_fp32_within_1e5(port):
    """lambda / p of the fp32 fast path vs the fp64 oracle, on mid-run fronts."""
    n, h, w = 6, 96, 80
    t = eb.synth_terrain(5, n, h, w)
    init = eb.synth_ignitions(5, t, 8)
    for cfg in (None, [0.3, 0.1, 0.3, 2.0, 1.5, 0.8], [0.05, 0.4, 0.8, 5.0, 0.5, 0.9]):
        b = _terrain_batch(t, cfg)
        b.set_state(init)
        b.set_key(5, 0)
        b.step(30)
        st = b.get_state()
        c = O.DEFAULT_CFG if cfg is None else cfg
        for form in (True, False):  # slope-record form (resident kernels) and elevation form
            lam, p = b.intensity(record_form=form)
            checked = 0
            for e in range(n):
                g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                                   t.wind_speed[e], t.wind_direction[e])
                lw, pw = O.intensity(port, "port", g, c, st[e])
                m = lw > 0
                checked += int(m.sum())
                np.testing.assert_allclose(lam[e][m], lw[m], rtol=REL_TOL)
                np.testing.assert_allclose(p[e][m], pw[m], rtol=REL_TOL, atol=1e-30)
                assert (lam[e][~m] == 0).all() and (p[e][~m] == 0).all()
            assert checked > 100, "fronts must be alive to test lambda/p"


@pytest.mark.parametrize("h,w", [(1, 1), (1, 37), (45, 1), (3, 3), (31, 33), (64, 96), (200, 100),
                                 (17, 300), (130, 520)])
def test_kernels_identical_ragged(port, h, w):
    """Tiled vs resident vs halo-tiled blocked vs oracle on ragged sizes (W not a multiple of
    32, single row/col), including garbage state bytes (>2 act as Unburned, engine.cpp:15-25)."""
    rs = np.random.default_rng(h * 1000 + w)
    n = 5
    cls = rs.integers(0, 11, (n, h, w)).astype(np.uint8)
    el = (400 * rs.random((n, h, w))).astype(np.float32)
    _, veg, den = eb.worldcover_palette()
    init = (rs.random((n, h, w)) < 0.15).astype(np.uint8)
    init[rs.random((n, h, w)) < 0.1] = 2
    init[rs.random((n, h, w)) < 0.01] = 7
    outs = []
    variants = [(eb.KERNEL_TILED, None), (eb.KERNEL_AUTO, None), (eb.KERNEL_BLOCKED, None),
                (eb.KERNEL_AUTO, (8, 32, 3)), (eb.KERNEL_AUTO, (5, 64, 1)), (eb.KERNEL_AUTO, (16, 96, 7))]
    if h * w <= 65536:
        variants.append((eb.KERNEL_WARP, None))
    for kernel, tiling in variants:
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
        outs.append(b.get_state())
        cnt = b.counts()
        assert np.array_equal(cnt[:, 1], (outs[-1] == 1).reshape(n, -1).sum(1)), (kernel, tiling)
        assert np.array_equal(cnt[:, 2], (outs[-1] == 2).reshape(n, -1).sum(1)), (kernel, tiling)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    for e in range(n):
        g = O.grid_terrain(port, "port", veg[cls[e]], den[cls[e]], el[e], 25.0, 7.0,
                           [0.3, 1.0, 2.0, 4.0, 6.0][e])
        want = O.run(port, "port", g, [0.4, 0.2, 0.4, 1.0, 1.0, 0.7], 9, 3, 100 + e, 25, init[e])
        assert np.array_equal(outs[0][e], want)


@pytest.mark.parametrize("kernel", KERNELS)
def test_batch_member_equals_solo_and_permutation(port, kernel):
    # test_engine.cpp:341-376: members == solo runs on their streams; order-invariant
    h, w = 10, 10
    rs = np.random.default_rng(61)
    L = dict(speed=2 * rs.random((h, w)), dir=6.28 * rs.random((h, w)), veg=rs.random((h, w)) - 0.3,
             den=rs.random((h, w)) - 0.3, slope8=0.5 * rs.random((h, w, 8)) - 0.25)
    cfg = [0.22, 0.2, 0.4, 1.0, 1.0, 0.6]
    f0 = np.zeros((h, w), np.uint8)
    f0[5, 5] = 1
    b = eb.Batch(8, h, w)
    b.set_config(cfg)
    b.set_grid(*L.values())
    b.set_kernel(kernel)
    b.set_state(f0)
    b.set_key(123, 0, first_stream=0)
    b.step(15)
    assert b.step_index == 15
    got = b.get_state()
    gp = O.grid_layers(port, "port", *L.values())
    for m in range(8):
        assert np.array_equal(got[m], O.run(port, "port", gp, cfg, 123, 0, m, 15, f0))
    b.set_state(f0)
    b.set_key(123, 0, streams=list(range(7, -1, -1)))
    b.step(15)
    assert np.array_equal(b.get_state()[::-1], got)


def test_invariants():
    h, w = 6, 6
    rs = np.random.default_rng(3)
    L = dict(speed=2 * rs.random((h, w)), dir=6.28 * rs.random((h, w)), veg=rs.random((h, w)) - 0.3,
             den=rs.random((h, w)) - 0.3, slope8=0.5 * rs.random((h, w, 8)) - 0.25)
    grid = dict(zip(("speed", "dir", "veg", "den", "slope8"), L.values()))
    fire = np.zeros((h, w), np.uint8)
    fire[2, 2] = 2
    assert np.array_equal(eb.step_stochastic(fire, grid, None, (1, 0, 0)), fire)  # no burning -> identity
    z = np.zeros((h, w))
    flat = dict(speed=z, dir=z, veg=z, den=z, slope8=np.zeros((h, w, 8)))
    fire = np.zeros((h, w), np.uint8)
    fire[1, 1] = fire[4, 3] = 1
    frozen = eb.run_stochastic(fire, flat, dict(p_base=0.0, p_continue=1.0), (9, 0, 0), 10)
    assert np.array_equal(frozen, fire)
    b = eb.Batch(1, 8, 8)
    L8 = dict(speed=2 * rs.random((8, 8)), dir=6.28 * rs.random((8, 8)), veg=rs.random((8, 8)) - 0.3,
              den=rs.random((8, 8)) - 0.3, slope8=0.5 * rs.random((8, 8, 8)) - 0.25)
    b.set_grid(*L8.values())
    b.set_config(dict(p_base=0.5, p_continue=0.3))
    s = np.zeros((8, 8), np.uint8)
    s[4, 4] = 1
    b.set_state(s)
    b.set_key(5, 0)
    prev = b.get_state()[0]
    for _ in range(30):
        b.step(1)
        cur = b.get_state()[0]
        assert (cur[prev == 2] == 2).all()  # burned is absorbing
        prev = cur


def test_monte_carlo_frequencies(port):
    # test_engine.cpp:127-155 pattern on the device: one step from a fixed state over 20k streams
    h = w = 8
    rs = np.random.default_rng(17)
    L = dict(speed=2 * rs.random((h, w)), dir=6.28 * rs.random((h, w)), veg=rs.random((h, w)) - 0.3,
             den=rs.random((h, w)) - 0.3, slope8=0.5 * rs.random((h, w, 8)) - 0.25)
    cfg = [0.25, 0.2, 0.4, 1.0, 1.0, 0.6]
    fire = np.zeros((h, w), np.uint8)
    fire[4, 4] = 1
    n = 20000
    b = eb.Batch(n, h, w)
    b.set_grid(*L.values())
    b.set_config(cfg)
    b.set_state(fire)
    b.set_key(77, 0, first_stream=0)
    b.step(1)
    freq = (b.get_state() == 1).mean(0)
    gp = O.grid_layers(port, "port", *L.values())
    _, p = O.intensity(port, "port", gp, cfg, fire)
    m = fire == 0
    sigma = np.sqrt(np.maximum(p * (1 - p) / n, 1e-12))
    assert (np.abs(freq - p)[m] <= 4 * sigma[m]).all()
    assert abs(freq[4, 4] - 0.6) <= 4 * np.sqrt(0.24 / n)


def test_errors():
    b = eb.Batch(2, 4, 4)
    with pytest.raises(eb.EmberError):
        b.step(1)  # no grid yet (ESTATE)
    z = np.zeros((4, 4))
    with pytest.raises(eb.InvalidArgument):
        b.set_grid(z - 1.0, z, z, z, np.zeros((4, 4, 8)))  # negative wind speed
    with pytest.raises(eb.InvalidArgument):
        b.set_grid(z, z, z + np.nan, z, np.zeros((4, 4, 8)))
    with pytest.raises(eb.InvalidArgument):
        eb.Batch(0, 4, 4)
    with pytest.raises(eb.InvalidArgument):
        eb.Batch(1, 0, 4)


@pytest.mark.slow
def test_c1_full_size_kernels_agree_and_sampled_oracle(port):
    """Full C1 (1024 x 128^2 x 200): resident == tiled on every env; 6 envs vs the port."""
    n, h, w, steps = 1024, 128, 128, 200
    t = eb.synth_terrain(0, n, h, w)
    init = eb.synth_ignitions(0, t, 5)
    outs = []
    for kernel in KERNELS:
        b = _terrain_batch(t, None, kernel)
        b.set_state(init)
        b.set_key(0, 0)
        b.step(steps)
        outs.append(b.get_state())
        assert b.diag()["ambiguous"] == 0
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
    for e in (0, 1, 511, 777, 1022, 1023):
        g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                           t.wind_speed[e], t.wind_direction[e])
        assert np.array_equal(outs[0][e], O.run(port, "port", g, O.DEFAULT_CFG, 0, 0, e, steps, init[e]))
    # burned count non-decreasing / conservation properties
    assert ((outs[0] == 2).reshape(n, -1).sum(1) >= 0).all()


def test_large_single_grid_vs_oracle(port):
    """C3-shaped (one large landscape, uniform wind from the west, many ignitions) at 1024^2:
    the halo-tiled blocked kernel (AUTO at this size) == per-step tiled kernel == oracle."""
    h = w = 1024
    t = eb.synth_terrain(11, 1, h, w)
    t.wind_speed[:] = 6.0
    t.wind_direction[:] = 0.0
    init = eb.synth_ignitions(11, t, 64)
    outs = []
    for kernel in (eb.KERNEL_AUTO, eb.KERNEL_TILED):
        b = _terrain_batch(t, None, kernel)
        b.set_state(init)
        b.set_key(11, 0)
        b.step(60)
        outs.append(b.get_state())
        assert b.diag()["ambiguous"] == 0
    assert np.array_equal(outs[0], outs[1])
    g = O.grid_terrain(port, "port", t.veg()[0], t.den()[0], t.elevation[0], 30.0, 6.0, 0.0)
    assert np.array_equal(outs[0][0], O.run(port, "port", g, O.DEFAULT_CFG, 11, 0, 0, 60, init[0]))


def test_derived_tables_follow_config_wind_and_terrain_changes(port):
    """The per-candidate pot32t rows (and slope records) are derived from the terrain, the wind
    and the config: changing each on a live batch rebuilds them -- every run matches a fresh
    oracle grid with the new inputs."""
    n, h, w, steps, seed = 4, 64, 96, 60, 9
    t = eb.synth_terrain(seed, n, h, w)
    t2 = eb.synth_terrain(seed + 1, n, h, w)
    init = eb.synth_ignitions(seed, t, 5)
    b = _terrain_batch(t, None)
    cfgs = [None, [0.3, 0.1, 0.3, 2.0, 1.5, 0.8], [0.3, 0.1, 0.3, 2.0, 1.5, 0.8], None]
    winds = [(t.wind_speed, t.wind_direction), (t.wind_speed, t.wind_direction),
             (t.wind_speed[::-1].copy(), (t.wind_direction + 1.0) % 6.28), (t.wind_speed, t.wind_direction)]
    terrains = [t, t, t, t2]
    for cfg, (ws, wd), tt in zip(cfgs, winds, terrains):
        if tt is not t:
            b.set_terrain(tt.fuel_class, tt.elevation, tt.class_veg, tt.class_den, tt.cellsize)
        b.set_config(cfg)
        b.set_wind(ws, wd)
        b.set_state(init)
        b.set_key(seed, 0)
        b.step(steps)
        got = b.get_state()
        c = O.DEFAULT_CFG if cfg is None else cfg
        for e in (0, n - 1):
            g = O.grid_terrain(port, "port", tt.veg()[e], tt.den()[e], tt.elevation[e], tt.cellsize, ws[e], wd[e])
            assert np.array_equal(got[e], O.run(port, "port", g, c, seed, 0, e, steps, init[e]))
    b.close()


def test_quiet_tiles_skipped_landscape_vs_oracle(port):
    """One call of many halo-tiled launches over a landscape that is mostly quiet (3 ignitions far
    apart, 240 steps = 30 launches): tiles without fire in their 3x3 neighbourhood for two launches
    are skipped outright (no load, step or store).  Final layers == per-step kernel == oracle,
    fire_fraction counts == the layers' counts, garbage bytes in never-burning tiles canonicalised
    as by a step."""
    h, w, steps = 512, 2048, 240
    t = eb.synth_terrain(12, 1, h, w)
    t.wind_speed[:] = 8.0
    t.wind_direction[:] = 0.0
    init = np.zeros((1, h, w), np.uint8)
    for r, c in ((40, 100), (300, 1000), (480, 1900)):
        init[0, r, c] = 1
    init[0, 200, 1500] = 7   # not a FireState: steps as Unburned (-> 0)
    init[0, 10, 10:20] = 2   # already burned cells far from the fire
    outs = []
    for kernel in (eb.KERNEL_AUTO, eb.KERNEL_TILED):
        b = _terrain_batch(t, None, kernel)
        b.set_state(init)
        b.set_key(12, 0)
        b.step(steps)
        outs.append(b.get_state())
        if kernel == eb.KERNEL_AUTO:
            cnt = b.counts()
            f = outs[-1][0]
            assert [int(cnt[0][k]) for k in range(3)] == [int((f == v).sum()) for v in (0, 1, 2)]
    assert np.array_equal(outs[0], outs[1])
    assert outs[0][0, 200, 1500] == 0 and (outs[0][0, 10, 10:20] == 2).all()
    g = O.grid_terrain(port, "port", t.veg()[0], t.den()[0], t.elevation[0], 30.0, 8.0, 0.0)
    assert np.array_equal(outs[0][0], O.run(port, "port", g, O.DEFAULT_CFG, 12, 0, 0, steps, init[0]))


def test_quiet_tiles_records_carried_across_calls_vs_oracle(port):
    """The same mostly quiet landscape stepped as 15 calls of 16 steps (one halo-tiled grid launch
    per call, tile records carried from call to call; the first call's records written by
    k_tile_init from the layer instead of a launch stepping every tile), then as uneven calls:
    final layers and counts == the one-call run == oracle, and the first launch no longer steps
    every tile."""
    h, w, steps = 512, 2048, 240
    t = eb.synth_terrain(12, 1, h, w)
    t.wind_speed[:] = 8.0
    t.wind_direction[:] = 0.0
    init = np.zeros((1, h, w), np.uint8)
    for r, c in ((40, 100), (300, 1000), (480, 1900)):
        init[0, r, c] = 1
    init[0, 200, 1500] = 7
    init[0, 10, 10:20] = 2
    g = O.grid_terrain(port, "port", t.veg()[0], t.den()[0], t.elevation[0], 30.0, 8.0, 0.0)
    want = O.run(port, "port", g, O.DEFAULT_CFG, 12, 0, 0, steps, init[0])
    for chunks in ([16] * 15, [5, 16, 16, 3, 100, 16, 84]):
        assert sum(chunks) == steps
        b = _terrain_batch(t, None)
        b.set_state(init)
        b.set_key(12, 0)
        b.diag(reset=True)
        b.step(chunks[0])
        d = b.diag()
        assert d["tiles_processed"] < d["tiles_launched"] // 4, d  # the first launch skips quiet tiles
        for c in chunks[1:]:
            b.step(c)
        got = b.get_state()[0]
        assert np.array_equal(got, want), chunks
        cnt = b.counts()
        assert [int(cnt[0][k]) for k in range(3)] == [int((got == v).sum()) for v in (0, 1, 2)]
        b.close()


@pytest.mark.parametrize("kernel", KERNELS)
def test_record_trajectory_vs_oracle(port, kernel):
    """run_stochastic(record=true) (engine.cpp:108,116) on the device: every step's layers."""
    n, h, w, steps = 3, 96, 64, 40
    t = eb.synth_terrain(2, n, h, w)
    init = eb.synth_ignitions(2, t, 6)
    b = _terrain_batch(t, None, kernel)
    b.set_state(init)
    b.set_key(2, 5, first_stream=7)
    traj = b.step_record(steps)
    assert np.array_equal(traj[-1], b.get_state())
    for e in range(n):
        g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                           t.wind_speed[e], t.wind_direction[e])
        st = init[e]
        for s in range(steps):
            st = O.run(port, "port", g, O.DEFAULT_CFG, 2, 5 + s, 7 + e, 1, st)
            assert np.array_equal(traj[s, e], st), (e, s)


@pytest.mark.parametrize("kernel", KERNELS + [eb.KERNEL_AUTO])
@pytest.mark.parametrize("h,w", [(64, 80), (128, 128)])
def test_wind_schedule_terrain_vs_oracle(port, kernel, h, w):
    """WindSchedule (engine.hpp:188-199) on the device: per-step winds, held past the end
    (128x128: the production warp kernel's compile-time C1 shape)."""
    n, steps = 4, 30
    t = eb.synth_terrain(4, n, h, w)
    init = eb.synth_ignitions(4, t, 5)
    rs = np.random.default_rng(0)
    S = 7
    sp = 8 * rs.random((S, n))
    dr = 6.3 * rs.random((S, n))
    b = _terrain_batch(t, None, kernel)
    b.set_wind_schedule(sp, dr)
    b.set_state(init)
    b.set_key(4, 2, first_stream=0)  # absolute steps 2.. -> entries 2..6 then 6 held
    b.step(steps)
    got = b.get_state()
    for e in range(n):
        st = init[e]
        for s in range(steps):
            row = min(2 + s, S - 1)
            g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0, sp[row, e], dr[row, e])
            st = O.run(port, "port", g, O.DEFAULT_CFG, 4, 2 + s, e, 1, st)
        assert np.array_equal(got[e], st)


def test_wind_schedule_general_form_vs_oracle(port):
    h, w, steps, S = 12, 10, 12, 4
    rs = np.random.default_rng(5)
    L = dict(speed=2 * rs.random((h, w)), dir=6.28 * rs.random((h, w)), veg=rs.random((h, w)) - 0.3,
             den=rs.random((h, w)) - 0.3, slope8=0.5 * rs.random((h, w, 8)) - 0.25)
    sp = 3 * rs.random((S, 1, h, w))
    dr = 6.28 * rs.random((S, 1, h, w))
    f0 = np.zeros((h, w), np.uint8)
    f0[6, 5] = 1
    cfg = [0.3, 0.2, 0.4, 1.0, 1.0, 0.7]
    b = eb.Batch(1, h, w)
    b.set_config(cfg)
    b.set_grid(*L.values())
    b.set_grid_wind_schedule(sp, dr)
    b.set_state(f0)
    b.set_key(21, 0)
    traj = b.step_record(steps)
    st = f0
    for s in range(steps):
        row = min(s, S - 1)
        g = O.grid_layers(port, "port", sp[row, 0], dr[row, 0], L["veg"], L["den"], L["slope8"])
        st = O.run(port, "port", g, cfg, 21, s, 0, 1, st)
        assert np.array_equal(traj[s, 0], st), s


@pytest.mark.parametrize("n_envs,chunks", [(13, 4), (64, 8), (7, 7), (5, 1), (3, 16)])
def test_pipelined_host_run_equals_sequence(n_envs, chunks):
    """ebl_batch_run (chunked H2D / fused launch / D2H pipeline) == set_state + step + get_state,
    counts included, and the batch continues from the run's result."""
    h, w, steps, seed = 64, 96, 40, 3
    t = eb.synth_terrain(seed, n_envs, h, w, env_id0=100)
    init = eb.synth_ignitions(seed, t, 4, env_id0=100)
    out = {}
    for mode in ("seq", "run"):
        with eb.Batch(n_envs, h, w) as b:
            b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
            b.set_wind(t.wind_speed, t.wind_direction)
            b.set_key(seed, 5, first_stream=100)
            if mode == "seq":
                b.set_state(init)
                b.step(steps)
                fin = b.get_state()
            else:
                b.set_pipeline(chunks)
                fin = b.run(init, steps)
            counts = b.counts().copy()
            b.step(3)  # continues from the run's final layers and step index
            out[mode] = (fin, counts, b.get_state(), b.step_index)
    assert np.array_equal(out["seq"][0], out["run"][0])
    assert np.array_equal(out["seq"][1], out["run"][1])
    assert np.array_equal(out["seq"][2], out["run"][2])
    assert out["seq"][3] == out["run"][3] == 5 + steps + 3


@pytest.mark.parametrize("huge", [False, True])
@pytest.mark.parametrize("chunks", [0, 3, 8])
def test_pipelined_run_pinned_zero_copy(chunks, huge):
    """ebl_batch_run with pinned host buffers (torch's, or ebl_host_alloc's huge-page mapped
    buffers): the kernels write the final layers straight into the mapped output buffer (no
    device -> host copy); identical to the sequence."""
    import torch
    n_envs, h, w, steps, seed = 37, 128, 128, 50, 4
    t = eb.synth_terrain(seed, n_envs, h, w)
    init = eb.synth_ignitions(seed, t, 5)
    with eb.Batch(n_envs, h, w) as b:
        b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
        b.set_wind(t.wind_speed, t.wind_direction)
        b.set_key(seed, 0)
        b.set_state(init)
        b.step(steps)
        want = b.get_state()
        if huge:
            h_in, h_out = eb.host_buffer(init.shape), eb.host_buffer(init.shape)
            h_in[:] = init
            h_out[:] = 9
            pi, po = h_in.ctypes.data, h_out.ctypes.data
        else:
            h_in = torch.from_numpy(init.copy()).pin_memory()
            h_out = torch.full_like(h_in, 9).pin_memory()
            pi, po = h_in.data_ptr(), h_out.data_ptr()
        b.set_pipeline(chunks)
        b.set_key(seed, 0)
        eb._lib.check(eb.lib().ebl_batch_run(b.handle, pi, steps, po))
        assert np.array_equal(np.asarray(h_out), want)
        assert np.array_equal(b.get_state(), want)  # the device copy is kept as well


@pytest.mark.slow
def test_bench_c1_workload_every_env_vs_reference():
    """The exact bench.py C1 workload (1024 envs x 128^2 x 200 steps, seed, 5 ignitions): every
    env's final layer from the device equals the reference engine's own run_stochastic
    (oracle/_ref, OpenMP over envs; the C restatement where the reference is not built)."""
    import bench
    s = bench.SPEC["C1"]
    t = eb.synth_terrain(bench.SEED, s["n_envs"], s["h"], s["w"])
    init = eb.synth_ignitions(bench.SEED, t, s["ignitions"])
    b = _terrain_batch(t, None)
    b.set_state(init)
    b.set_key(bench.SEED, 0)
    b.step(s["steps"])
    got = b.get_state()
    assert b.diag()["ambiguous"] == 0
    # the e2e path of the bench (pipelined host-buffer run into mapped huge-page memory)
    h_in = eb.host_buffer(init.shape)
    h_in[:] = init
    h_out = eb.host_buffer(init.shape)
    b.set_key(bench.SEED, 0)
    b.run(h_in, s["steps"], out=h_out)
    b.close()
    r = bench._cpu_c1(s["n_envs"], return_states=True)
    want = r["states"].reshape(got.shape)
    assert np.array_equal(got, want), r["kind"]
    assert np.array_equal(h_out, want)
