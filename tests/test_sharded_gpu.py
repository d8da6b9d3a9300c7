"""C3 path: one landscape row-sharded into G shards with light-cone halos (here G shards on
device 0; on G GPUs the halo copies go peer-to-peer) is bit-identical to the unsharded run
and to the oracle, because the RNG cell index stays global (engine.cpp:17)."""
import numpy as np
import pytest

import paper_2512_06102_b200 as eb
from oracle import oracle as O
from paper_2512_06102_b200.sharded import ShardedLandscape

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("g,halo", [(1, 8), (2, 8), (3, 4), (4, 8), (5, 2), (10, 4)])
def test_sharded_equals_unsharded(port, g, halo, fused):
    h, w, steps, seed = 300, 200, 45, 3
    t = eb.synth_terrain(seed, 1, h, w)
    t.wind_speed[:] = 6.0
    t.wind_direction[:] = 0.0  # "from the west": pushes east (kernel.hpp:24)
    init = eb.synth_ignitions(seed, t, 16)
    full = eb.Batch(1, h, w)
    full.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    full.set_wind(t.wind_speed, t.wind_direction)
    full.set_state(init)
    full.set_key(seed, 0, first_stream=0)
    full.step(steps)
    want = full.get_state()[0]
    sh = ShardedLandscape(t, g, halo=halo, fused=fused)
    sh.set_state(init[0])
    sh.set_key(seed, 0, 0)
    sh.step(steps - 7)
    sh.step(7)  # a second call continues from the first (halo rows already exchanged)
    got = sh.get_state()
    counts = sum(b.counts()[0] for b in sh.batches) if fused else None
    if fused:  # band rows only: the shards' counts add up to the landscape's
        assert counts[:3].tolist() == [int((want == k).sum()) for k in range(3)]
    assert np.array_equal(got, want), np.argwhere(got != want)[:5]
    gp = O.grid_terrain(port, "port", t.veg()[0], t.den()[0], t.elevation[0], 30.0, 6.0, 0.0)
    assert np.array_equal(want, O.run(port, "port", gp, O.DEFAULT_CFG, seed, 0, 0, steps, init[0]))


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("direction", [0.0, 90.0, 270.0])
@pytest.mark.parametrize("g", [2, 4, 6, 9])  # 9 > kMaxShardLaunch: per-shard launches and events
def test_fire_across_shard_boundaries_small_tiles(g, direction, fused):
    """The tile records travel with the halo rows -- fused: a burning tile enqueues the neighbour
    shard's tiles next to the rows it stores there; per-rank form: the halo-row copies mark the
    records they reach (ember_warp.cu k_mark_halo).  Fires lit on every band boundary, small
    16 x 64 tiles with 4-row light cones (so many quiet tiles sit next to the halo rows), several
    calls -- equal to the unsharded run, and tiles really are skipped."""
    h, w, seed = 480, 256, 11
    t = eb.synth_terrain(seed, 1, h, w)
    t.wind_speed[:] = 8.0
    t.wind_direction[:] = direction
    init = eb.synth_ignitions(seed, t, 4)
    burnable = t.class_veg[t.fuel_class[0]] > -1.0
    for k in range(1, g):  # both sides of every band edge
        edge = k * h // g
        for r in (edge - 2, edge - 1, edge, edge + 1):
            for c in range(7, w, 61):
                if burnable[r, c]:
                    init[0, r, c] = 1
    full = eb.Batch(1, h, w)
    full.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    full.set_wind(t.wind_speed, t.wind_direction)
    full.set_state(init)
    full.set_key(seed, 0, first_stream=0)
    sh = ShardedLandscape(t, g, halo=4, fused=fused)
    for b in sh.batches:
        b.set_tiling(16, 64, 4)
        b.diag(reset=True)
    sh.set_state(init[0])
    sh.set_key(seed, 0, 0)
    for n in (37, 60, 83):
        full.step(n)
        sh.step(n)
        want = full.get_state()[0]
        got = sh.get_state()
        assert np.array_equal(got, want), (n, np.argwhere(got != want)[:5])
        if fused:  # (the per-rank form's counts include its halo rows)
            tot = sum(b.counts()[0] for b in sh.batches)
            assert tot[:3].tolist() == [int((want == k).sum()) for k in range(3)]
    run = sum(b.diag()["tiles_processed"] for b in sh.batches)
    launched = sum(b.diag()["tiles_launched"] for b in sh.batches)
    assert run < 0.9 * launched, (run, launched)


def test_rows_device_roundtrip():
    import torch
    b = eb.Batch(2, 40, 64)
    rs = np.random.default_rng(0)
    st = rs.integers(0, 3, (2, 40, 64)).astype(np.uint8)
    b.set_state(st)
    buf = torch.empty((2, 5, 64), dtype=torch.uint8, device="cuda:0")
    eb._lib.check(eb.lib().ebl_batch_rows_device(b.handle, 10, 5, buf.data_ptr(), 0))
    assert np.array_equal(buf.cpu().numpy(), st[:, 10:15])
    buf.fill_(2)
    eb._lib.check(eb.lib().ebl_batch_rows_device(b.handle, 30, 5, buf.data_ptr(), 1))
    st[:, 30:35] = 2
    assert np.array_equal(b.get_state(), st)


@pytest.mark.slow
def test_c3_full_size_shards_equal_unsharded():
    """BASELINE C3 at full size (one 16384 x 16384 landscape, wind 6 from the west, 64 ignitions,
    500 steps): 4 fused row shards == the unsharded run, bit for bit, and the size-independent
    properties hold -- cells conserved, burnt only grows, every burnt or burning cell is burnable
    or an ignition, the shard counts add up to the landscape's."""
    h = w = 16384
    steps = 500
    t = eb.synth_terrain(0, 1, h, w)
    t.wind_speed[:] = 6.0
    t.wind_direction[:] = 0.0
    init = eb.synth_ignitions(0, t, 64)
    full = eb.Batch(1, h, w)
    full.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    full.set_wind(t.wind_speed, t.wind_direction)
    full.set_state(init)
    full.set_key(0, 0, first_stream=0)
    full.step(200)
    mid = full.get_state()[0]
    full.step(steps - 200)
    want = full.get_state()[0]
    cnt = full.counts()[0]
    full.close()
    assert cnt[:3].tolist() == [int((want == k).sum()) for k in range(3)]
    assert cnt[:3].sum() == h * w
    assert ((want == 2) | (mid != 2)).all(), "a burnt cell never changes"
    assert (want != 0).sum() >= (mid != 0).sum() >= (init[0] != 0).sum()
    burnable = t.class_veg[t.fuel_class[0]] > -1.0
    assert ((want == 0) | burnable | (init[0] != 0)).all()
    sh = ShardedLandscape(t, 4, halo=8, fused=True)
    sh.set_state(init[0])
    sh.set_key(0, 0, 0)
    sh.step(steps)
    got = sh.get_state()
    assert np.array_equal(got, want)
    total = sum(b.counts()[0] for b in sh.batches)
    assert total[:3].tolist() == cnt[:3].tolist()


def _c3_landscape(size, seed=0):
    t = eb.synth_terrain(seed, 1, size, size)
    t.wind_speed[:] = 6.0
    t.wind_direction[:] = 0.0  # "from the west"
    return t, eb.synth_ignitions(seed, t, 64)


def test_c3_4096_500_steps_quiet_tiles_vs_reference():
    """The C3 geometry at 4096^2 x 500 steps (C3 generator, wind 6 from the west, 64 ignitions):
    the production path (a tile-record init, then 32 work-list launches of 16 steps, quiet tiles
    skipped outright) equals
    the reference's own run_stochastic (oracle/_ref, OpenMP) bit for bit, counts included; then
    fused row shards G = 2 / 4 / 8 (quiet tiles kept across the chunks, the boundary tiles' records
    exchanged with the halo rows)
    and the per-rank form (step + halo-row copies, records carried across calls) equal it too.
    Every run really skips tiles (tile statistics)."""
    R = O.ref()
    if R is None:
        pytest.skip("reference not built (oracle/_ref)")
    size, steps, seed = 4096, 500, 0
    t, init = _c3_landscape(size, seed)
    full = eb.Batch(1, size, size)
    full.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    full.set_wind(t.wind_speed, t.wind_direction)
    full.set_state(init)
    full.set_key(seed, 0, first_stream=0)
    full.diag(reset=True)
    full.step(steps)
    got = full.get_state()[0]
    cnt = full.counts()[0]
    d = full.diag()
    full.close()
    # the tile-record init, 32 step launches (+ the counts reduction)
    assert d["launches"] in (33, 34) and d["ambiguous"] == 0
    assert 0 < d["tiles_processed"] < 0.8 * d["tiles_launched"], d
    g = O.grid_terrain(R, "ref", t.veg()[0], t.den()[0], t.elevation[0], 30.0, 6.0, 0.0)
    out = np.empty_like(init[0])
    rc = R.ref_run_stochastic(g.h, O.ptr(O.cfg_array(O.DEFAULT_CFG)), seed, 0, 0, steps, 1,
                              O.ptr(np.ascontiguousarray(init[0])), O.ptr(out))
    assert rc == 0
    assert np.array_equal(got, out), np.argwhere(got != out)[:5]
    assert cnt[:3].tolist() == [int((out == k).sum()) for k in range(3)]
    for G, halo in ((2, 8), (4, 16), (8, 16)):  # 16: the library's default light cone
        sh = ShardedLandscape(t, G, halo=halo, fused=True)
        sh.set_state(init[0])
        sh.set_key(seed, 0, 0)
        for b in sh.batches:
            b.diag(reset=True)
        sh.step(steps)
        assert np.array_equal(sh.get_state(), out), G
        tot = sum(b.counts()[0] for b in sh.batches)
        assert tot[:3].tolist() == cnt[:3].tolist()
        run = sum(b.diag()["tiles_processed"] for b in sh.batches)
        launched = sum(b.diag()["tiles_launched"] for b in sh.batches)
        assert run < 0.8 * launched, (G, run, launched)
    sh = ShardedLandscape(t, 4, halo=16, fused=False)   # per-rank form: step(16) + halo copies
    sh.set_state(init[0])
    sh.set_key(seed, 0, 0)
    for b in sh.batches:
        b.diag(reset=True)
    sh.step(steps)
    assert np.array_equal(sh.get_state(), out)
    run = sum(b.diag()["tiles_processed"] for b in sh.batches)
    launched = sum(b.diag()["tiles_launched"] for b in sh.batches)
    assert run < 0.8 * launched, (run, launched)


def test_shards_across_two_devices_fused_peer_stores():
    """The fused NVLink halo exchange across devices: 4 shards alternating over GPUs 0 and 1 (peer
    stores into the neighbour's layer, stream-event ordering across devices) equal the unsharded
    run.  Runs only where two GPUs are visible (the round's boxes have one)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    h, w, steps, seed = 600, 512, 120, 5
    t = eb.synth_terrain(seed, 1, h, w)
    t.wind_speed[:] = 6.0
    t.wind_direction[:] = 0.0
    init = eb.synth_ignitions(seed, t, 24)
    full = eb.Batch(1, h, w)
    full.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    full.set_wind(t.wind_speed, t.wind_direction)
    full.set_state(init)
    full.set_key(seed, 0, first_stream=0)
    full.step(steps)
    want = full.get_state()[0]
    sh = ShardedLandscape(t, 4, devices=[0, 1, 0, 1], halo=8, fused=True)
    sh.set_state(init[0])
    sh.set_key(seed, 0, 0)
    sh.step(steps)
    assert np.array_equal(sh.get_state(), want)
    assert torch.cuda.current_device() == 0  # the library restores the caller's device
