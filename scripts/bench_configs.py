"""Throughput of every BASELINE config on one B200 (bench.py is the C1 headline; this covers
C0, C2, C3, C4 the same way): CUDA events on the launch stream, warm-up, L2 flushed between
timed iterations, the reference / port CPU path timed beside it on a bounded sample.
Prints one JSON line per config; `--out` appends them to a file.

  python scripts/bench_configs.py [--configs c0,c2,c3,c4] [--out profiles/r01_configs.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_06102_b200 as eb  # noqa: E402
from oracle import oracle as O  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
FLUSH = None
STREAM = None  # the stream every timed batch launches on (set in main)


def flush_l2():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    FLUSH.zero_()


def timed(fn, iters, warmup=3):
    """fn() issues work on the current torch stream; returns per-iteration ms (events)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(iters):
        flush_l2()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(STREAM)
        fn()
        e.record(STREAM)
        e.synchronize()
        out.append(s.elapsed_time(e))
    return out


def line(cfg, metric, value, unit, ms, alg_bytes, extra=None):
    d = {"config": cfg, "metric": metric, "value": value, "unit": unit, "ms_per_step": ms,
         "roofline": {"bound": "hbm", "alg_bytes_per_step": alg_bytes,
                      "achieved_GBps": alg_bytes / (ms * 1e-3) / 1e9,
                      "frac": alg_bytes / (ms * 1e-3) / 1e9 / PEAK, "peak": PEAK}}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)
    return d


def bench_c0(iters):
    h = w = 64
    z = np.zeros((h, w))
    stream = STREAM  # a real stream: the legacy default (0) would make the batch use its own
    b = eb.Batch(1, h, w, stream=stream.cuda_stream)
    b.set_grid(z, z, z, z, np.zeros((h, w, 8)))
    fire = np.zeros((1, h, w), np.uint8)
    fire[0, 32, 32] = 1
    dev = torch.from_numpy(fire).cuda()

    def run():
        eb._lib.check(eb.lib().ebl_batch_set_state_device(b.handle, dev.data_ptr()))
        b.set_key(0, 0)
        b.step(100)
    ms = timed(run, iters)
    t = float(np.median(ms))
    # end to end: the one-shot run_stochastic signature (host buffers, tables built inside)
    grid = dict(speed=z, dir=z, veg=z, den=z, slope8=np.zeros((h, w, 8)))
    eb.run_stochastic(fire[0], grid, None, (0, 0, 0), 100)
    t0 = time.perf_counter()
    for _ in range(iters):
        eb.run_stochastic(fire[0], grid, None, (0, 0, 0), 100)
    e2e = (time.perf_counter() - t0) / iters * 1e3
    R = O.ref()
    g = O.grid_layers(R, "ref", z, z, z, z, np.zeros((h, w, 8)))
    t0 = time.perf_counter()
    for _ in range(20):
        O.run(R, "ref", g, O.DEFAULT_CFG, 0, 0, 0, 100, fire[0])
    cpu = (time.perf_counter() - t0) / 20 * 1e3
    cells = h * w * 100
    return line("C0: 64x64 flat, 100 steps, 1 env", "cell-updates/sec", cells / (t * 1e-3), "cell-updates/s",
                t, cells * 10, {"e2e_ms": e2e, "e2e_value": cells / (e2e * 1e-3),
                                "cpu_baseline": {"kind": "reference", "ms": cpu, "value": cells / (cpu * 1e-3),
                                                 "cores": 1, "sample": "the full C0 run, Exec::serial"},
                                "note": "latency-bound: one 100-step launch of a 4096-cell env"})


def bench_c2(iters):
    n, h, w, steps = 16384, 64, 64, 256
    t = eb.synth_terrain(0, n, h, w)
    env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=None, ignitions=5, max_steps=256)
    env.reset(0)
    torch.cuda.synchronize()

    def roll():
        eb._lib.check(eb.lib().ebl_rl_rollout(env.batch.handle, steps, None, None))
    # the rollout runs on the batch's own stream: time it with host sync around (device-bound)
    for _ in range(2):
        roll()
        env.batch.sync()
    ts = []
    for _ in range(iters):
        flush_l2()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        roll()
        env.batch.sync()
        ts.append((time.perf_counter() - t0) * 1e3)
    ms = float(np.median(ts))
    env_steps = n * steps
    # per-step API (actions from the device policy, reward/done to host each step)
    t0 = time.perf_counter()
    for _ in range(32):
        env.step(None)
    step_ms = (time.perf_counter() - t0) / 32 * 1e3
    # port baseline: the C restatement of the same tanker step, 8 envs x 64 steps (grids and
    # SpreadTables built before the timed region, as the reference env builds its tables once)
    P = O.port()
    tc = O.TankerCfg(5, 256, 1)
    envs = []
    for e in range(8):
        g = O.grid_terrain(P, "port", t.veg()[e], t.den()[e], t.elevation[e], 30.0, t.wind_speed[e],
                           t.wind_direction[e])
        pot, gam = O.tables(P, "port", g, O.DEFAULT_CFG, h * w)
        s = O.TankerSt()
        f = np.zeros((h, w), np.uint8)
        wt = np.zeros((h, w), np.uint8)
        P.ebo_tanker_reset(g.h, tc, 0, e, 0, s, O.ptr(f), O.ptr(wt))
        envs.append((e, g, pot, gam, s, f, wt))
    rw = np.zeros(1, np.float32)
    dn = np.zeros(1, np.uint8)
    t0 = time.perf_counter()
    cnt = 0
    for e, g, pot, gam, s, f, wt in envs:
        for _ in range(64):
            a = P.ebo_tanker_policy(0, e, s, h * w)
            P.ebo_tanker_step(g.h, O.ptr(pot), O.ptr(gam), 0.6, tc, 0, e, a, s, O.ptr(f), O.ptr(wt),
                              O.ptr(rw), O.ptr(dn))
            cnt += 1
    cpu_s = time.perf_counter() - t0
    return line("C2: 16384 envs x 64x64 tanker RL, 256 steps, device random (x,y) policy, auto-reset",
                "env-steps/sec", env_steps / (ms * 1e-3), "env-steps/s", ms, env_steps * 40973,
                {"cell_updates_per_sec": env_steps * h * w / (ms * 1e-3),
                 "per_step_api": {"ms_per_step": step_ms, "env_steps_per_sec": n / (step_ms * 1e-3),
                                  "note": "ebl_rl_step per step, reward/done read back each step"},
                 "cpu_baseline": {"kind": "port", "value": cnt / cpu_s, "unit": "env-steps/s", "cores": 1,
                                  "sample": "8 envs x 64 steps of the C restatement of the tanker step"}})


def bench_c3(iters, size):
    h = w = size
    t0 = time.perf_counter()
    t = eb.synth_terrain(0, 1, h, w)
    t.wind_speed[:] = 6.0
    t.wind_direction[:] = 0.0
    init = eb.synth_ignitions(0, t, 64)
    host_setup_ms = (time.perf_counter() - t0) * 1e3
    stream = STREAM
    b = eb.Batch(1, h, w, stream=stream.cuda_stream)
    # environment construction on the device: same layers, bit for bit
    b.synth_terrain(0)
    b.sync()
    t0 = time.perf_counter()
    b.synth_terrain(0)
    b.set_wind([6.0], [0.0])
    b.synth_ignitions(0, 64)
    b.sync()
    dev_setup_ms = (time.perf_counter() - t0) * 1e3
    fc, el = b.get_terrain()
    assert np.array_equal(fc, t.fuel_class) and np.array_equal(b.get_state(), init)
    del fc, el
    dev = torch.from_numpy(init).cuda()
    steps = 500

    def run():
        eb._lib.check(eb.lib().ebl_batch_set_state_device(b.handle, dev.data_ptr()))
        b.set_key(0, 0)
        b.step(steps)
    ms = float(np.median(timed(run, iters, warmup=1)))
    cells = h * w * steps
    # reference baseline on a bounded sample: 2048^2 x 20 steps, OpenMP (Exec::parallel)
    R = O.ref()
    hs = 2048
    g = O.grid_terrain(R, "ref", t.veg()[0][:hs, :hs], t.den()[0][:hs, :hs], t.elevation[0][:hs, :hs], 30.0, 6.0, 0.0)
    st = np.ascontiguousarray(init[0][:hs, :hs])
    out = np.empty_like(st)
    t0 = time.perf_counter()
    R.ref_run_stochastic(g.h, O.ptr(O.cfg_array(O.DEFAULT_CFG)), 0, 0, 0, 20, 1, O.ptr(st), O.ptr(out))
    cpu = time.perf_counter() - t0
    return line(f"C3: one {h}x{w} landscape, wind 6 from the west, 64 ignitions, 500 steps, 1 GPU",
                "cell-updates/sec", cells / (ms * 1e-3), "cell-updates/s", ms, cells * 10,
                {"launches_per_run": -(-steps // 8),
                 "env_construction_ms": {"host": host_setup_ms, "device": dev_setup_ms,
                                         "note": "C1 generator + 64 ignitions at 16384^2; bit-identical"},
                 "cpu_baseline": {"kind": "reference", "value": hs * hs * 20 / cpu, "unit": "cell-updates/s",
                                  "cores": R.ref_max_threads(),
                                  "sample": "2048^2 corner x 20 steps, run_stochastic Exec::parallel (incl. tables)"}})


def bench_c4(iters):
    n, h, w, steps = 256, 128, 128, 100
    t = eb.synth_terrain(4, n, h, w)
    init = eb.synth_ignitions(4, t, 5)
    b = eb.Batch(n, h, w)
    b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed, t.wind_direction)
    b.set_config(None)
    mask = (np.random.default_rng(0).random((n, h, w)) < 0.2).astype(np.float64)
    b.set_state(init)
    b.det_set_state_from_fire()
    b.det_forward(1, record=True)  # builds the tables once (setup, not timed)
    b.det_set_mask(mask)  # the calibration target: resident across iterations (as ebl_calibrate)

    def run():
        b.det_set_state_from_fire()
        b.det_forward(steps, record=True)
        b.det_loss_grad(None, 0.0, 1.0, 1)
    for _ in range(2):
        run()
    ts = []
    for _ in range(iters):
        flush_l2()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run()
        ts.append((time.perf_counter() - t0) * 1e3)
    ms = float(np.median(ts))
    cell_steps = n * h * w * steps
    P = O.port()
    g = O.grid_terrain(P, "port", t.veg()[0], t.den()[0], t.elevation[0], 30.0, t.wind_speed[0], t.wind_direction[0])
    lo, g6 = O._D(), np.empty(6)
    t0 = time.perf_counter()
    P.ebo_det_loss_grad(g.h, O.ptr(O.cfg_array(O.DEFAULT_CFG)), steps, O.ptr(init[0]),
                        O.ptr(np.ascontiguousarray(mask[0])), 0.0, 1.0, 1, lo, O.ptr(g6))
    cpu = time.perf_counter() - t0
    return line("C4: 256 envs x 128x128, 100 deterministic steps + loss + reverse-mode gradient (fp64)",
                "cell-steps/sec", cell_steps / (ms * 1e-3), "cell-steps/s (fwd+bwd)", ms, cell_steps * 80,
                {"note": "host-timed end to end: state from the fire layers, trajectory record, loss against the "
                         "resident target, reverse-mode gradient, loss + gradient readback",
                 "cpu_baseline": {"kind": "port", "value": h * w * steps / cpu, "unit": "cell-steps/s", "cores": 1,
                                  "sample": "1 env: Dual<6> forward-mode run_deterministic + loss (C restatement)"}})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c0,c2,c3,c4")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--c3-size", type=int, default=16384)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    global STREAM
    STREAM = torch.cuda.Stream()
    res = []
    for c in a.configs.split(","):
        if c == "c0":
            res.append(bench_c0(a.iters))
        elif c == "c2":
            res.append(bench_c2(a.iters))
        elif c == "c3":
            res.append(bench_c3(a.iters, a.c3_size))
        elif c == "c4":
            res.append(bench_c4(a.iters))
    if a.out:
        with open(a.out, "a") as f:
            for r in res:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
