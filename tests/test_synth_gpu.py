"""Environment construction on the device vs the host/oracle paths.

* the C1 generator on the device == the host generator (ebl_synth_terrain), bit for bit;
* device ignitions == host ignitions;
* fuel_from_landcover / grid_from_rasters on the device == the reference (oracle/_ref) and the
  numpy restatement pinned against it (tests/test_oracle_pin.py);
* DEM nodata (NaN elevation) slopes: every kernel bit-exact vs the port, which is pinned vs the
  reference's slope_from_dem on nodata rasters."""
import numpy as np
import pytest

import paper_2512_06102_b200 as eb
from oracle import oracle as O
from test_oracle_pin import landcover_restated

pytestmark = pytest.mark.gpu

KERNELS = [eb.KERNEL_TILED, eb.KERNEL_RESIDENT, eb.KERNEL_BLOCKED, eb.KERNEL_WARP, eb.KERNEL_AUTO]
WORLDCOVER = {10: (0.4, 0.3), 20: (0.25, 0.1), 30: (0.15, -0.1), 40: (0.0, -0.2), 50: (-0.8, -0.8),
              60: (-0.7, -0.6), 70: (-1.0, -1.0), 80: (-1.0, -1.0), 90: (-0.4, -0.3),
              95: (-0.2, -0.1), 100: (-0.3, -0.4)}


@pytest.mark.parametrize("seed,env0,n,h,w", [(0, 0, 3, 128, 128), (7, 100, 2, 37, 53), (1, 0, 1, 2, 3),
                                             (2, 5, 4, 5, 300), (3, 9, 1, 200, 77), (4, 0, 2, 2, 2),
                                             (5, 1, 1, 513, 260)])
def test_device_synth_equals_host(seed, env0, n, h, w):
    t = eb.synth_terrain(seed, n, h, w, env_id0=env0)
    b = eb.Batch(n, h, w)
    b.synth_terrain(seed, env_id0=env0)
    fc, el = b.get_terrain()
    assert np.array_equal(fc, t.fuel_class)
    assert np.array_equal(el.view(np.uint32), t.elevation.view(np.uint32))
    if h * w >= 11:
        assert len(np.unique(fc)) > 1
    # ignitions: same cells as the host redraw loop
    for count in (0, 1, 5, min(h * w, 40)):
        placed = b.synth_ignitions(seed, count, env_id0=env0)
        want = eb.synth_ignitions(seed, t, count, env_id0=env0)
        assert np.array_equal(b.get_state(), want)
        assert placed == int((want == 1).sum())


def test_device_synth_steps_like_host_terrain(port):
    """Device-built env == host-built env through 150 steps; wind per env is the host's."""
    n, h, w, seed = 6, 128, 128, 3
    t = eb.synth_terrain(seed, n, h, w)
    b = eb.Batch(n, h, w)
    b.synth_terrain(seed)
    b.synth_ignitions(seed, 5)
    b.set_key(seed, 0)
    b.step(150)
    got = b.get_state()
    init = eb.synth_ignitions(seed, t, 5)
    for e in (0, n - 1):
        g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                           t.wind_speed[e], t.wind_direction[e])
        assert np.array_equal(got[e], O.run(port, "port", g, O.DEFAULT_CFG, seed, 0, e, 150, init[e]))
    assert b.diag()["ambiguous"] == 0


def test_device_synth_deterministic_mode():
    """The deterministic mode's host tables read the device-built terrain back (lazy fetch)."""
    n, h, w = 2, 40, 40
    t = eb.synth_terrain(9, n, h, w)
    outs = []
    for dev in (False, True):
        b = eb.Batch(n, h, w)
        if dev:
            b.synth_terrain(9)
        else:
            b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
            b.set_wind(t.wind_speed, t.wind_direction)
        fire = np.zeros((n, h, w), np.uint8)
        fire[:, 20, 20] = 1
        b.set_state(fire)
        b.det_set_state_from_fire()
        b.det_forward(20)
        outs.append(b.det_get_state())
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


def _landcover_case(seed, h, w, unknown=True):
    rs = np.random.default_rng(seed)
    el = (250 * rs.random((h, w))).astype(np.float32)
    el[rs.random((h, w)) < 0.03] = np.nan
    codes = list(WORLDCOVER) + ([7] if unknown else [])
    lc = rs.choice(codes, (h, w)).astype(np.int32)
    return el, lc


@pytest.mark.parametrize("h,w", [(33, 47), (1, 5), (128, 128)])
def test_landcover_vs_reference(port, h, w):
    el, lc = _landcover_case(h * 7 + w, h, w)
    nodata_code = -9999
    lc[lc == 20] = nodata_code
    lcf = lc.astype(np.float64)
    lcf[lc == nodata_code] = np.nan
    fb = (0.05, -0.05)
    b = eb.Batch(1, h, w)
    b.set_landcover(lc, el, WORLDCOVER, fallback=fb, nodata_code=nodata_code)
    fc, el_dev = b.get_terrain()
    pal_v, pal_d = _palette(WORLDCOVER, fb)
    want_v, want_d = landcover_restated(lcf, el, WORLDCOVER, fb)
    assert np.array_equal(pal_v[fc[0]], want_v) and np.array_equal(pal_d[fc[0]], want_d)
    assert np.array_equal(el_dev[0].view(np.uint32), el.view(np.uint32))
    R = O.ref()
    if R is not None:
        _, rv, rd = O.grid_from_rasters(R, el, lcf, WORLDCOVER, fallback=fb)
        assert np.array_equal(pal_v[fc[0]], rv) and np.array_equal(pal_d[fc[0]], rd)
    # stepping on the mapped terrain (nodata slopes included) == the port
    fire = np.zeros((h, w), np.uint8)
    fire[h // 2, w // 2] = 1
    b.set_wind([3.0], [1.0])
    b.set_state(fire)
    b.set_key(4, 0)
    b.step(30)
    g = O.grid_terrain(port, "port", want_v, want_d, el, 30.0, 3.0, 1.0)
    assert np.array_equal(b.get_state()[0], O.run(port, "port", g, O.DEFAULT_CFG, 4, 0, 0, 30, fire))


def _palette(table, fallback):
    codes = sorted(table)
    v = [table[c][0] for c in codes] + ([fallback[0]] if fallback else []) + [-1.0]
    d = [table[c][1] for c in codes] + ([fallback[1]] if fallback else []) + [-1.0]
    return np.array(v), np.array(d)


def test_landcover_errors():
    el, lc = _landcover_case(5, 16, 16)
    b = eb.Batch(1, 16, 16)
    with pytest.raises(eb._lib.FileError, match="no entry for landcover code 7"):
        b.set_landcover(lc, el, WORLDCOVER)
    with pytest.raises(eb._lib.InvalidArgument, match="must lie in"):
        b.set_landcover(lc, el, {10: (1.5, 0.0)}, fallback=(0, 0))
    with pytest.raises(eb._lib.InvalidArgument, match="fallback"):
        b.set_landcover(lc, el, WORLDCOVER, fallback=(0, 2.0))
    # repeated codes: the last entry wins (FuelTable::set overwrites)
    b2 = eb.Batch(1, 4, 4)
    lc2 = np.full((4, 4), 10, np.int32)
    codes = np.array([10, 10], np.int32)
    veg = np.array([0.1, 0.7])
    den = np.array([0.2, -0.3])
    el2 = np.zeros((4, 4), np.float32)
    eb._lib.check(eb.lib().ebl_batch_set_landcover(b2.handle, 1, lc2.ctypes.data, el2.ctypes.data, 0, 0, 2,
                                                   codes.ctypes.data, veg.ctypes.data, den.ctypes.data,
                                                   0, 0.0, 0.0, 30.0))
    fc, _ = b2.get_terrain()
    assert (fc == 0).all()
    fire = np.zeros((4, 4), np.uint8)
    fire[1, 1] = 1
    b2.set_state(fire)
    b2.set_key(0, 0)
    b2.step(3)  # palette (0.7, -0.3) in force: just must run


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("h,w", [(96, 80), (128, 128), (64, 64), (300, 260)])
def test_dem_nodata_all_kernels_vs_port(port, kernel, h, w):
    """DEM nodata (NaN elevation: slope 0 toward/from the cell, geodata.cpp:214,220) on every
    kernel, including the production AUTO/WARP path with its pot32t rows at the compile-time
    128x128 / 64x64 shapes and the halo-tiled geometry (300x260 > 65536 cells)."""
    if kernel == eb.KERNEL_RESIDENT and h * w > 65536:
        pytest.skip("resident kernel needs a whole env in shared memory")
    n, seed = 3, 12
    t = eb.synth_terrain(seed, n, h, w)
    rs = np.random.default_rng(1)
    t.elevation[rs.random(t.elevation.shape) < 0.05] = np.nan
    t.elevation[:, h // 2 - 2:h // 2 + 2, :] = np.nan  # a nodata band across the fire path
    init = eb.synth_ignitions(seed, t, 6)
    b = eb.Batch(n, h, w)
    b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed, t.wind_direction)
    b.set_config([0.3, 0.2, 0.4, 2.0, 1.0, 0.7])
    b.set_kernel(kernel)
    b.set_state(init)
    b.set_key(seed, 0)
    b.step(90)
    got = b.get_state()
    for e in range(n):
        g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                           t.wind_speed[e], t.wind_direction[e])
        want = O.run(port, "port", g, [0.3, 0.2, 0.4, 2.0, 1.0, 0.7], seed, 0, e, 90, init[e])
        assert np.array_equal(got[e], want), f"env {e}"
    assert b.diag()["ambiguous"] == 0
