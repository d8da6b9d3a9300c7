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
    for _ in range(2):
        b = _batch(t, None)
        b.set_state(init)
        b.det_set_state_from_fire()
        b.det_forward(steps, record=True)
        outs.append(b.det_loss_grad(mask, 0.0, 1.0, 1))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert np.isfinite(outs[0][1]).all() and (np.abs(outs[0][1]).sum(1) > 0).all()
