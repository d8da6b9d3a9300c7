"""Device snapshot rendering (ebl_batch_snapshot_text) against the reference's texts
(tests/golden/snapshots.json) and the C restatement of serialize_snapshot."""
import json
import os

import numpy as np
import pytest

import paper_2512_06102_b200 as eb
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "snapshots.json")))


@pytest.mark.parametrize("case", GOLD["serialize"], ids=lambda c: f"{c['h']}x{c['w']}")
def test_batch_snapshot_matches_reference(case):
    h, w = case["h"], case["w"]
    fire = np.array(case["fire"], np.uint8).reshape(1, h, w)
    with eb.Batch(1, h, w) as b:
        b.set_state(fire)
        agents = [case["agent"]] if case["agent"] else None
        assert b.snapshot_text(steps=[case["step"]], agents=agents) == case["text"]


def test_batch_snapshots_of_a_recorded_trajectory():
    """A trajectory recorded on the device (step_record's device form) rendered in one call, one
    snapshot per (step, env), equals the port's texts; garbage bytes render as '?'."""
    import ctypes as C
    import torch
    n, h, w, steps, seed = 3, 20, 45, 6, 2
    t = eb.synth_terrain(seed, n, h, w)
    init = eb.synth_ignitions(seed, t, 4)
    init[1, 0, :3] = [5, 9, 255]
    with eb.Batch(n, h, w) as b:
        b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
        b.set_wind(t.wind_speed, t.wind_direction)
        b.set_key(seed, 0)
        b.set_state(init)
        text0 = b.snapshot_text()
        want0 = "".join(O.snapshot_text(O.port(), "port", init[e], 0).decode() for e in range(n))
        assert text0 == want0
        traj = torch.empty((steps, n, h, w), dtype=torch.uint8, device="cuda")
        eb._lib.check(eb.lib().ebl_step_batch_record(b.handle, steps, C.c_void_p(traj.data_ptr()), 1))
        torch.cuda.synchronize()
        st = np.repeat(np.arange(1, steps + 1), n)
        ag = np.array([[e, e + 1, 7] if e != 1 else [-1, 0, 0] for _ in range(steps) for e in range(n)])
        text = b.snapshot_text(traj.data_ptr(), steps * n, steps=st, agents=ag)
        tr = traj.cpu().numpy()
        want = "".join(O.snapshot_text(O.port(), "port", tr[k, e], k + 1, None if e == 1 else (e, e + 1, 7)).decode()
                       for k in range(steps) for e in range(n))
        assert text == want
        layer, step, agent = eb.parse_snapshot(want.split("emberline-snapshot")[3].join(["emberline-snapshot", ""]))
        assert step == 1 and agent == (2, 3, 7)
