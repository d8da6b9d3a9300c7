"""Deterministic mode (engine.hpp:147-245) and the C4 reverse-mode gradient on the device vs
the oracle: the fp64 forward (run_deterministic<double>) and the forward-mode Dual<6> gradient
(restated in oracle/ember_oracle.c and pinned bitwise to the reference in test_oracle_pin.py).
Bar: gradients within 1e-4 relative (BASELINE C4); fp64 state within 1e-9 relative."""
import numpy as np
import pytest

import paper_2512_06102_b200 as eb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GRAD_RTOL = 1e-4  # BASELINE C4 bar


def _batch(t, cfg):
    n, h, w = t.fuel_class.shape
    b = eb.Batch(n, h, w)
    b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, t.cellsize)
    b.set_wind(t.wind_speed, t.wind_direction)
    b.set_config(cfg)
    return b


def _hidden_target(t, init, seed, steps):
    """Target burn masks from the same model under hidden parameters drawn from a seed
    (the run_self_calibration pattern, calibrate.cpp:203-215): threshold(p_burn + p_bd, 0.5)."""
    rs = np.random.default_rng(seed)
    theta = [0.12 * rs.uniform(0.5, 1.5), 0.2 * rs.uniform(0.5, 1.5), 0.4 * rs.uniform(0.5, 1.5),
             1.0 * rs.uniform(0.5, 1.5), 1.0 * rs.uniform(0.5, 1.5), min(0.95, 0.6 * rs.uniform(0.5, 1.5))]
    b = _batch(t, theta)
    b.set_state(init)
    b.det_set_state_from_fire()
    b.det_forward(steps, record=False)
    _, burn, bd = b.det_get_state()
    mask = ((burn.astype(np.float64) + bd) >= 0.5).astype(np.float64)
    mask[:, 0, 0] = 1.0  # validate_target: at least one burned cell
    return theta, mask


def test_forward_matches_fp64_oracle(port):
    n, h, w, steps = 6, 64, 48, 50
    t = eb.synth_terrain(21, n, h, w)
    init = eb.synth_ignitions(21, t, 4)
    cfg = [0.2, 0.15, 0.3, 1.2, 0.9, 0.7]
    b = _batch(t, cfg)
    b.set_state(init)
    b.det_set_state_from_fire()
    b.det_forward(steps, record=False)
    un, burn, bd = b.det_get_state()
    for e in range(n):
        g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                           t.wind_speed[e], t.wind_direction[e])
        u = (init[e] == 0).astype(np.float64)
        bu = (init[e] == 1).astype(np.float64)
        bdd = (init[e] == 2).astype(np.float64)
        port.ebo_det_run(g.h, O.ptr(O.cfg_array(cfg)), steps, O.ptr(u), O.ptr(bu), O.ptr(bdd))
        # the reference's own fp64 arithmetic: equal up to CUDA-vs-glibc exp ulps at x >= 2^-20
        np.testing.assert_allclose(burn[e], bu, rtol=1e-9, atol=1e-15)
        np.testing.assert_allclose(un[e], u, rtol=1e-9, atol=1e-15)
        np.testing.assert_allclose(bd[e], bdd, rtol=1e-9, atol=1e-15)
        assert np.abs(un[e] + burn[e] + bd[e] - 1).max() < 1e-12  # simplex (test_engine.cpp:215-233)


@pytest.mark.parametrize("bce_w,mse_w,pool", [(0.0, 1.0, 1), (1.0, 1.0, 4)])
def test_c4_gradient_vs_dual_oracle(port, bce_w, mse_w, pool):
    """C4: 128x128, 100 steps, loss = MSE (pool 1) [+ the reference's default BCE + pooled
    variant]; reverse-mode device gradient vs the Dual<6> forward-mode oracle."""
    n, h, w, steps, seed = 4, 128, 128, 100, 4
    t = eb.synth_terrain(seed, n, h, w)
    init = eb.synth_ignitions(seed, t, 5)
    _, mask = _hidden_target(t, init, seed, steps)
    cfg0 = [0.12, 0.2, 0.4, 1.0, 1.0, 0.6]  # theta0 = SimConfig{}
    b = _batch(t, cfg0)
    b.set_state(init)
    b.det_set_state_from_fire()
    b.det_forward(steps, record=True)
    loss, grad = b.det_loss_grad(mask, bce_w, mse_w, pool)
    for e in range(n):
        g = O.grid_terrain(port, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0,
                           t.wind_speed[e], t.wind_direction[e])
        lo, g6 = O._D(), np.empty(6)
        port.ebo_det_loss_grad(g.h, O.ptr(O.cfg_array(cfg0)), steps, O.ptr(init[e]),
                               O.ptr(np.ascontiguousarray(mask[e])), bce_w, mse_w, pool, lo, O.ptr(g6))
        assert loss[e] == pytest.approx(lo.value, rel=GRAD_RTOL)
        scale = np.abs(g6).max()
        np.testing.assert_allclose(grad[e], g6, rtol=GRAD_RTOL, atol=GRAD_RTOL * 1e-2 * scale)


def test_c4_full_batch_runs_and_is_deterministic():
    """The full C4 batch (256 x 128^2 x 100) through forward + backward twice: identical bits."""
    n, h, w, steps, seed = 256, 128, 128, 100, 4
    t = eb.synth_terrain(seed, n, h, w)
    init = eb.synth_ignitions(seed, t, 5)
    _, mask = _hidden_target(t, init, seed, steps)
    outs = []
    for resident in (False, True):  # per-call mask, then the det_set_mask target
        b = _batch(t, None)
        b.set_state(init)
        b.det_set_state_from_fire()
        b.det_forward(steps, record=True)
        if resident:
            with pytest.raises(eb.EmberError, match="ebl_det_set_mask"):
                b.det_loss_grad(None)  # no resident target yet
            b.det_set_mask(mask)
        outs.append(b.det_loss_grad(None if resident else mask, 0.0, 1.0, 1))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert np.isfinite(outs[0][1]).all() and (np.abs(outs[0][1]).sum(1) > 0).all()


def test_c4_all_256_envs_vs_reference_dual():
    """BASELINE C4 at full size: every one of the 256 envs (128^2, 100 steps, MSE vs the
    hidden-parameter target) -- the device's reverse-mode gradient against the reference's own
    run_deterministic<Dual<6>> + loss (oracle/_ref, OpenMP over envs; the pattern of
    tests/test_calibrate.cpp:276-298), within 1e-4 relative; losses within 1e-9."""
    R = O.ref()
    if R is None:
        pytest.skip("reference not built (oracle/_ref)")
    n, h, w, steps, seed = 256, 128, 128, 100, 4
    t = eb.synth_terrain(seed, n, h, w)
    init = eb.synth_ignitions(seed, t, 5)
    _, mask = _hidden_target(t, init, seed, steps)
    b = _batch(t, None)
    b.set_state(init)
    b.det_set_state_from_fire()
    b.det_forward(steps, record=True)
    loss, grad = b.det_loss_grad(mask, 0.0, 1.0, 1)
    grids = [O.grid_terrain(R, "ref", t.veg()[e], t.den()[e], t.elevation[e], 30.0, t.wind_speed[e],
                            t.wind_direction[e]) for e in range(n)]
    hs = (O._P * n)(*[g.h for g in grids])
    want_l = np.empty(n)
    want_g = np.empty((n, 6))
    secs = R.ref_loss_grad_envs(hs, n, O.ptr(O.cfg_array(O.DEFAULT_CFG)), steps, O.ptr(np.ascontiguousarray(init)),
                                O.ptr(np.ascontiguousarray(mask)), 0.0, 1.0, 1, O.ptr(want_l), O.ptr(want_g), 0)
    assert secs >= 0, R.ref_last_error()
    np.testing.assert_allclose(loss, want_l, rtol=1e-9, atol=0)
    for e in range(n):
        scale = np.abs(want_g[e]).max()
        np.testing.assert_allclose(grad[e], want_g[e], rtol=GRAD_RTOL, atol=GRAD_RTOL * 1e-2 * scale,
                                   err_msg=f"env {e}")
    # the batch gradient the calibration step consumes (fixed-order sum over envs)
    np.testing.assert_allclose(grad.sum(0), want_g.sum(0), rtol=GRAD_RTOL)


def _calib_case(seed=3, h=20, w=17):
    rs = np.random.default_rng(seed)
    L = dict(speed=np.full((h, w), 1.5), dir=np.full((h, w), 0.9), veg=rs.random((h, w)) * 0.6 + 0.1,
             den=rs.random((h, w)) * 0.5 + 0.1, slope8=0.4 * rs.random((h, w, 8)) - 0.2)
    fire = np.zeros((h, w), np.uint8)
    fire[h // 2, w // 2] = 1
    planes = [(fire == k).astype(np.float64) for k in (0, 1, 2)]
    return L, planes


@pytest.mark.parametrize("kw", [dict(), dict(bce_weight=0.0, mse_weight=1.0, pool=1),
                                dict(optimize=[1, 0, 1, 1, 0, 1])])
def test_calibrate_on_device_matches_reference_loop(port, kw):
    """calibrate (calibrate.cpp:104-167) with the device rollout/loss/gradient on a general
    GridState vs the oracle's Dual<6> loop (itself bitwise equal to the reference)."""
    L, planes = _calib_case()
    h, w = L["veg"].shape
    gp = O.grid_layers(port, "port", *L.values())
    un, bu, bd = [p.copy() for p in planes]
    port.ebo_det_run(gp.h, O.ptr(O.cfg_array([0.22, 0.15, 0.3, 0.8, 1.1, 0.7])), 12, O.ptr(un), O.ptr(bu), O.ptr(bd))
    mask = ((bu + bd) >= 0.5).astype(np.float64)
    init = [0.15, 0.2, 0.25, 1.1, 0.9, 0.6]
    okw = {("bce_w" if k == "bce_weight" else "mse_w" if k == "mse_weight" else k): v for k, v in kw.items()}
    rc, lh, thh, best, bl = O.calibrate(port, "port", gp, planes, mask, 12, 10, init, **okw)
    assert rc == 0
    b = eb.Batch(1, h, w)
    b.set_grid(*L.values())
    res = b.calibrate(*planes, mask, 12, iterations=10, init_theta=init, **kw)
    np.testing.assert_allclose(res["loss_history"], lh, rtol=1e-9)
    np.testing.assert_allclose(res["theta_history"], thh, rtol=1e-9, atol=1e-12)
    assert res["best_loss"] == pytest.approx(bl, rel=1e-9)
    with pytest.raises(eb.InvalidArgument):
        b.calibrate(*planes, mask * 0, 12, iterations=1)  # no burned cell in the target


def test_det_general_form_gradient_vs_dual(port):
    """The general (per-cell layers) form of the adjoint vs Dual<6>, 30 steps, BCE + pooled MSE."""
    L, _ = _calib_case(seed=8, h=33, w=29)
    h, w = L["veg"].shape
    fire = np.zeros((h, w), np.uint8)
    fire[5, 7] = fire[20, 20] = 1
    rs = np.random.default_rng(1)
    mask = (rs.random((h, w)) < 0.3).astype(np.float64)
    cfg = [0.25, 0.1, 0.35, 0.9, 1.2, 0.65]
    b = eb.Batch(1, h, w)
    b.set_grid(*L.values())
    b.set_config(cfg)
    b.set_state(fire)
    b.det_set_state_from_fire()
    b.det_forward(30, record=True)
    loss, grad = b.det_loss_grad(mask, 1.0, 1.0, 4)
    gp = O.grid_layers(port, "port", *L.values())
    lo, g6 = O._D(), np.empty(6)
    port.ebo_det_loss_grad(gp.h, O.ptr(O.cfg_array(cfg)), 30, O.ptr(fire), O.ptr(mask), 1.0, 1.0, 4, lo, O.ptr(g6))
    assert loss[0] == pytest.approx(lo.value, rel=1e-12)
    np.testing.assert_allclose(grad[0], g6, rtol=1e-9, atol=1e-14)


def test_c4_env_shards_sum_to_the_whole():
    """C4 sharded by env (one process per GPU in production): two halves of the batch, run as
    separate batches, give per-env losses / gradients identical to the whole batch, and their
    fixed-order sum equals the whole batch's (distributed.reduce_loss_grad's contract)."""
    from paper_2512_06102_b200.distributed import env_range, sum_loss_grad
    n, h, w, steps, seed = 6, 48, 48, 25, 4
    t = eb.synth_terrain(seed, n, h, w)
    init = eb.synth_ignitions(seed, t, 4)
    mask = (np.random.default_rng(1).random((n, h, w)) < 0.2).astype(np.float64)

    def run(ids):
        b = eb.Batch(len(ids), h, w)
        b.set_terrain(t.fuel_class[ids], t.elevation[ids], t.class_veg, t.class_den, 30.0)
        b.set_wind(t.wind_speed[ids], t.wind_direction[ids])
        b.set_state(init[ids])
        b.det_set_state_from_fire()
        b.det_forward(steps, record=True)
        return b.det_loss_grad(mask[ids])

    loss_all, grad_all = run(list(range(n)))
    parts = [run(list(range(*env_range(r, 2, n)))) for r in range(2)]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), loss_all)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), grad_all)
    assert sum_loss_grad(loss_all, grad_all)[0] == sum_loss_grad(
        np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))[0]


@pytest.mark.parametrize("shared_grid", [False, True])
def test_device_built_tables_bit_identical_to_host(shared_grid):
    """The terrain-form SpreadTables built on the device (cached fp64 slopes + the restated libm
    exp, ember_exp.cuh) equal the host build bit for bit: identical fp64 forward states, losses
    and gradients after config changes (the calibration loop's pattern), with DEM nodata cells."""
    n, h, w, steps, seed = 6, 128, 128, 40, 8
    t = eb.synth_terrain(seed, n, h, w)
    t.elevation[:, 50:53, :] = np.nan
    init = eb.synth_ignitions(seed, t, 5)
    mask = (np.random.default_rng(1).random((n, h, w)) < 0.3).astype(np.float64)
    res = {}
    for dev in (0, 1):
        b = eb.Batch(n, h, w)
        if shared_grid:  # one terrain, per-env winds: tables per env over grid 0
            b.set_terrain(t.fuel_class[:1], t.elevation[:1], t.class_veg, t.class_den, 30.0)
        else:
            b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
        b.set_wind(t.wind_speed, t.wind_direction)
        eb._lib.check(eb.lib().ebl_batch_set_det_tables(b.handle, dev))
        out = []
        for cfg in ([0.12, 0.2, 0.4, 1.0, 1.0, 0.6], [0.2, 0.1, 0.7, 2.7, 0.8, 0.75], [0.05, 0.3, 0.2, -1.3, 1.4, 0.5]):
            b.set_config(cfg)
            b.set_state(init)
            b.det_set_state_from_fire()
            b.det_forward(steps, record=True)
            out.append(b.det_get_state())
            out.append(b.det_loss_grad(mask, 0.0, 1.0, 1))
        res[dev] = out
        b.close()
    for x, y in zip(res[0], res[1]):
        for p, q in zip(x, y):
            assert np.array_equal(np.asarray(p).view(np.uint64), np.asarray(q).view(np.uint64))


@pytest.mark.parametrize("steps", [1, 2, 37])
def test_recorded_forward_p_bd_after_the_run_bit_identical(steps):
    """The recorded forward leaves p_bd out of its steps and replays p_bd += p_burn(t)(1 - p_continue)
    (engine.hpp:164-167) over the recorded p_burn planes after the run (k_det_bd_run): its final
    state, p_bd included, is bit-identical to the unrecorded forward's (odd and even step counts:
    the state buffers end on either side of the ping-pong)."""
    n, h, w = 3, 64, 48
    t = eb.synth_terrain(5, n, h, w)
    init = eb.synth_ignitions(5, t, 4)
    out = []
    for record in (False, True):
        b = _batch(t, [0.2, 0.15, 0.3, 1.2, 0.9, 0.7])
        b.set_state(init)
        b.det_set_state_from_fire()
        b.det_forward(steps, record=record)
        out.append(b.det_get_state())
        b.close()
    for p, q in zip(*out):
        assert np.array_equal(np.asarray(p).view(np.uint64), np.asarray(q).view(np.uint64))
