"""Benchmark of the batched CA fire-spread step (BASELINE.json metric) on every BASELINE config.

  python bench.py [--config C1|C0|C2|C3|C4] [--impl ours|reference] [--scaling weak|strong]
                  [--gpus N --steps K --warmup W]

Default: C1 (configs[1], the config the headline metric is quoted on), N=1.  One bench "step" is
one pass of the hot path over one batch of synthetic inputs:

  C0  1 env 64x64 flat, uniform fuel, calm, centre ignition: a 100-step run (4.1e5 cell-updates)
  C1  1024 envs of 128x128, per-env seeded landcover/elevation/wind, 5 ignitions: a 200-step run
      of every env (3.36e9 cell-updates, counted densely as emberline_main.cpp:432-433)
  C2  16384 envs of 64x64 air-tanker RL (device random (x,y) policy, 3x3 drop, auto-reset):
      256 RL steps of every env (4.19e6 env-steps)
  C3  one 16384x16384 landscape, wind 6 from the west, 64 ignitions: a 500-step run
      (1.34e11 cell-updates); N>1: row bands per rank, 16-row halos exchanged every 16 steps
  C4  256 envs of 128x128, 100 deterministic fp64 steps + MSE loss + reverse-mode gradient of
      the 6 SimConfig parameters (4.19e8 cell-steps, forward + backward)

value      device throughput, inputs resident in HBM, CUDA events on the launch stream, L2
           flushed (256 MiB write) between timed iterations, max over ranks.
e2e        the same metric through the public C-ABI with HOST buffers (pinned), the host<->device
           copies of each step's inputs and results inside the timed region.
roofline   the dominant kernel: C1 against the SM issue rate (the kernel keeps the state in
           shared memory for all 200 steps, so HBM does not bind), with the HBM
           figures (algorithmic bytes of SURVEY §8(d) and ncu DRAM bytes) beside it; C0/C2/C3/C4
           against the measured HBM copy bandwidth at SURVEY §8(d)'s algorithmic bytes.
cpu_baseline  the reference's own code (oracle/_ref = /root/reference/proj compiled in place, or
           the C restatement where the reference has no such path) on this host's cores, a
           bounded sample of the same workload (rank 0, N=1).

Multi-GPU (torchrun, one process per GPU, NCCL): C1/C2/C4 shard envs by global env id with no
data-path collective ("weak": each rank its own full batch; "strong": the batch split across
ranks); C3 shards rows ("strong": one landscape).  `--impl reference` runs only the reference
CPU arm (rank 0; other ranks exit 0) with the same metric and config.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 0
SPEC = {
    "C0": dict(n_envs=1, h=64, w=64, steps=100, metric="cell-updates/sec", unit="cell-updates/s",
               workload="C0: 1 env 64x64, flat, uniform fuel (veg=den=0), calm, ignition at (32,32), "
                        "100 CA steps, SimConfig{}, RngKey{0,0,0}"),
    "C1": dict(n_envs=1024, h=128, w=128, steps=200, ignitions=5, metric="cell-updates/sec",
               unit="cell-updates/s",
               workload="C1: 1024 envs x 128x128, per-env value-noise landcover (11 WorldCover classes) "
                        "+ fractal elevation 0-500 m + wind U(0,10)/U(0,2pi), 5 ignitions, 200 CA steps"),
    "C2": dict(n_envs=16384, h=64, w=64, steps=256, ignitions=5, metric="env-steps/sec", unit="env-steps/s",
               workload="C2: 16384 envs x 64x64 air-tanker RL, C1 terrain generator, device random (x,y) "
                        "policy, 3x3 extinguish+wet, reward -(newly ignited), done at 0 burning or 256 "
                        "steps, auto-reset; 256 RL steps per bench step"),
    "C3": dict(n_envs=1, h=16384, w=16384, steps=500, ignitions=64, metric="cell-updates/sec",
               unit="cell-updates/s",
               workload="C3: one 16384x16384 landscape, C1 generator, wind 6 m/s from the west, "
                        "64 ignitions, 500 CA steps"),
    "C4": dict(n_envs=256, h=128, w=128, steps=100, ignitions=5, metric="cell-steps/sec",
               unit="cell-steps/s (forward + backward)",
               workload="C4: 256 envs x 128x128, 100 deterministic fp64 steps from the fire layers, "
                        "MSE loss vs a resident target mask, reverse-mode gradient of the 6 SimConfig "
                        "parameters"),
}
# SURVEY §8(d) algorithmic bytes: 10 per cell-update (stochastic), 40,973 per C2 env-step,
# 80 per C4 cell-step (value + gradient)
ALG_BYTES = {"C0": 10, "C1": 10, "C2": 40973, "C3": 10, "C4": 80}


def config_json(cfg: str, world: int, scaling: str) -> dict:
    """The workload description, identical in both arms (the implementation goes in `impl`)."""
    s = SPEC[cfg]
    per_rank = s["n_envs"] if scaling == "weak" or cfg in ("C0", "C3") else -(-s["n_envs"] // world)
    glob = s["n_envs"] * (world if scaling == "weak" and cfg not in ("C0", "C3") else 1)
    return {"workload": s["workload"], "global_batch": glob, "envs_per_rank": per_rank,
            "grid": [s["h"], s["w"]], "steps_per_run": s["steps"],
            "parallelism": (f"row-sharded x{world}" if cfg == "C3" else f"env-sharded x{world}"),
            "l2": "flushed between timed iterations (256 MiB write)",
            "seed": SEED}


def rank_envs(cfg: str, rank: int, world: int, scaling: str):
    """(first global env id, number of envs) of this rank.  Weak: every rank its own full batch
    (ids rank*n ..); strong: the batch split in contiguous id ranges."""
    n = SPEC[cfg]["n_envs"]
    if scaling == "weak":
        return rank * n, n
    lo = rank * n // world
    return lo, (rank + 1) * n // world - lo


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_counters(key: str):
    """Per-launch ncu counters of the dominant kernel (profiles/ncu_counters.json, written from an
    `ncu --set full` capture of this build); None when absent or for another kernel build."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_counters.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ================================================================================================
# CPU arms (the reference compiled in place, oracle/_ref; the C restatement where the reference
# has no such path).  Inputs come from the oracle's restatement of the input generator, pinned
# bit-for-bit to the product's (tests/test_oracle_pin.py): the product library is never loaded.
# ================================================================================================
def _cpu_c1(n_envs, h=128, w=128, steps=200, threads=0, return_states=False):
    from oracle import oracle as O
    R = O.ref()
    kind = "reference" if R is not None else "port"
    L = R if R is not None else O.port()
    t = O.SynthTerrain(SEED, n_envs, h, w)
    init = t.ignitions(SPEC["C1"]["ignitions"])
    grids = [O.grid_terrain(L, "ref" if R is not None else "port", t.veg()[e], t.den()[e], t.elevation[e],
                            30.0, t.wind_speed[e], t.wind_direction[e]) for e in range(n_envs)]
    handles = (O._P * n_envs)(*[g.h for g in grids])
    states = np.ascontiguousarray(init.copy())
    streams = np.arange(n_envs, dtype=np.uint64)
    fn = L.ref_run_envs if R is not None else L.ebo_run_envs
    secs = fn(handles, n_envs, O.ptr(O.cfg_array(O.DEFAULT_CFG)), SEED, O.ptr(streams), steps, O.ptr(states),
              threads)
    cores = (R.ref_max_threads() if R is not None else os.cpu_count()) if threads <= 0 else threads
    return dict(seconds=secs, units=n_envs * h * w * steps, kind=kind, cores=cores,
                sample=f"{n_envs} of the C1 envs x {steps} steps: run_stochastic(Exec::serial) per env "
                       f"(tables built inside, as the reference does), OpenMP over envs",
                states=states if return_states else None)


def _cpu_c0(reps):
    from oracle import oracle as O
    R = O.ref()
    h = w = 64
    z = np.zeros((h, w))
    g = O.grid_layers(R, "ref", z, z, z, z, np.zeros((h, w, 8)))
    fire = np.zeros((h, w), np.uint8)
    fire[32, 32] = 1
    out = np.empty_like(fire)
    t0 = time.perf_counter()
    for _ in range(reps):
        R.ref_run_stochastic(g.h, O.ptr(O.cfg_array(O.DEFAULT_CFG)), 0, 0, 0, 100, 1, O.ptr(fire), O.ptr(out))
    secs = time.perf_counter() - t0
    return dict(seconds=secs, units=reps * h * w * 100, kind="reference", cores=R.ref_max_threads(),
                sample=f"{reps} full C0 runs: run_stochastic(Exec::parallel), tables built inside")


def _cpu_c2(n_envs, steps=64):
    """The reference's own RL step path: FireSuppressionEnv (rl_env.cpp:125-210) on the C2 grid
    (64x64, 5 ignitions, SimConfig{} spread, 256-step cap; uniform fuel and flat terrain -- the
    reference env has no terrain or tanker action), random_policy, OpenMP over envs."""
    from oracle import oracle as O
    R = O.ref()
    cfg = O.EnvCfg()
    R.ref_env_preset(0, C.byref(cfg))
    cfg.height = cfg.width = 64
    cfg.ignition_count = 5
    cfg.max_episode_steps = 256
    for i, v in enumerate(O.DEFAULT_CFG):
        cfg.spread[i] = float(v)
    n = C.c_longlong()
    rs = C.c_double()
    secs = R.ref_env_batch(C.byref(cfg), n_envs, SEED, 0, steps, 0, C.byref(n), C.byref(rs))
    return dict(seconds=secs, units=n.value, kind="reference", cores=R.ref_max_threads(),
                sample=f"{n_envs} envs x {steps} steps of FireSuppressionEnv::step (64x64, reference "
                       "semantics: agent move + valve, uniform fuel), random_policy, OpenMP over envs")


def _cpu_c2_tanker(n_envs, steps=64):
    """The C restatement of the C2 tanker env itself (same semantics as the device path)."""
    from oracle import oracle as O
    t = O.SynthTerrain(SEED, n_envs, 64, 64)
    r = O.tanker_run_envs(t, np.arange(n_envs), O.DEFAULT_CFG, SEED, steps)
    return dict(seconds=r["seconds"], units=n_envs * steps, kind="port", cores=os.cpu_count(),
                sample=f"{n_envs} C2 envs x {steps} tanker steps (C restatement, tables prebuilt), "
                       "OpenMP over envs")


def _cpu_c3(size=4096, steps=10):
    from oracle import oracle as O
    R = O.ref()
    t = O.SynthTerrain(SEED, 1, size, size)
    init = t.ignitions(SPEC["C3"]["ignitions"])
    g = O.grid_terrain(R, "ref", t.veg()[0], t.den()[0], t.elevation[0], 30.0, 6.0, 0.0)
    out = np.empty_like(init[0])
    t0 = time.perf_counter()
    R.ref_run_stochastic(g.h, O.ptr(O.cfg_array(O.DEFAULT_CFG)), SEED, 0, 0, steps, 1, O.ptr(init[0]), O.ptr(out))
    secs = time.perf_counter() - t0
    return dict(seconds=secs, units=size * size * steps, kind="reference", cores=R.ref_max_threads(),
                sample=f"a {size}x{size} landscape of the C3 generator x {steps} steps: "
                       "run_stochastic(Exec::parallel) incl. its SpreadTables build (the reference's "
                       "16384^2 layout needs ~65 GB of host memory)")


def _cpu_c4(n_envs, steps=100):
    from oracle import oracle as O
    R = O.ref()
    h = w = 128
    t = O.SynthTerrain(4, n_envs, h, w)
    init = t.ignitions(SPEC["C4"]["ignitions"])
    mask = (np.random.default_rng(0).random((n_envs, h, w)) < 0.2).astype(np.float64)
    grids = [O.grid_terrain(R, "ref", t.veg()[e], t.den()[e], t.elevation[e], 30.0, t.wind_speed[e],
                            t.wind_direction[e]) for e in range(n_envs)]
    hs = (O._P * n_envs)(*[g.h for g in grids])
    loss = np.empty(n_envs)
    grad = np.empty((n_envs, 6))
    secs = R.ref_loss_grad_envs(hs, n_envs, O.ptr(O.cfg_array(O.DEFAULT_CFG)), steps, O.ptr(init),
                                O.ptr(mask), 0.0, 1.0, 1, O.ptr(loss), O.ptr(grad), 0)
    return dict(seconds=secs, units=n_envs * h * w * steps, kind="reference", cores=R.ref_max_threads(),
                sample=f"{n_envs} C4 envs x {steps} steps: run_deterministic<Dual<6>> + loss per env "
                       "(calibrate.cpp:144-146), OpenMP over envs")


def cpu_sample(cfg: str, target_s: float):
    """One bounded sample of the config's workload on the CPU, sized to ~target_s seconds."""
    if cfg == "C0":
        probe = _cpu_c0(2)
        return _cpu_c0(max(2, int(2 * target_s / max(probe["seconds"], 1e-4))))
    if cfg == "C1":
        probe = _cpu_c1(16)
        return _cpu_c1(int(max(16, min(SPEC["C1"]["n_envs"], 16 * target_s / max(probe["seconds"], 1e-3)))))
    if cfg == "C2":
        probe = _cpu_c2(64, 16)
        return _cpu_c2(int(max(64, min(SPEC["C2"]["n_envs"], 64 * target_s / max(probe["seconds"] * 4, 1e-3)))))
    if cfg == "C3":
        probe = _cpu_c3(1024, 4)
        steps = int(max(2, min(100, 4 * target_s / max(probe["seconds"] * 16, 1e-3))))
        return _cpu_c3(4096, steps)
    if cfg == "C4":
        probe = _cpu_c4(8, 10)
        return _cpu_c4(int(max(8, min(SPEC["C4"]["n_envs"], 8 * target_s / max(probe["seconds"] * 10, 1e-3)))))
    raise ValueError(cfg)


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    cfg = args.config
    s = SPEC[cfg]
    target = {"C0": 3.0, "C1": 4.0, "C2": 4.0, "C3": 6.0, "C4": 6.0}[cfg]
    for _ in range(args.warmup if cfg in ("C0", "C1") else 1):
        cpu_sample(cfg, 0.5)
    runs = [cpu_sample(cfg, target) for _ in range(args.steps)]
    value = sum(r["units"] for r in runs) / sum(r["seconds"] for r in runs)
    r0 = runs[0]
    line = {"metric": s["metric"], "value": value, "unit": s["unit"], "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(r["seconds"] for r in runs) / len(runs),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_json(cfg, world, args.scaling),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": s["unit"], "cores": r0["cores"], "kind": r0["kind"],
                             "sample": r0["sample"] + " (per bench step)"},
            "e2e": {"value": value, "unit": s["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if cfg == "C2":
        tk = _cpu_c2_tanker(256)
        line["cpu_port_same_semantics"] = {"value": tk["units"] / tk["seconds"], "unit": s["unit"],
                                           "cores": tk["cores"], "kind": "port", "sample": tk["sample"]}
    print(json.dumps(line), flush=True)
    return 0


# ================================================================================================
# GPU arm
# ================================================================================================
class Ctx:
    def __init__(self, args, rank, world, local):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.args, self.rank, self.world, self.local = args, rank, world, local
        self.dist_on = world > 1
        torch.cuda.set_device(local)
        if self.dist_on:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        self.dev = f"cuda:{local}"
        self.stream = torch.cuda.Stream()
        self.flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=self.dev)  # > 126 MB L2

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.dist_on:
            self.dist.barrier()

    def flush(self):
        with self.torch.cuda.stream(self.stream):
            self.flush_buf.zero_()

    def max_over_ranks(self, x: float) -> float:
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        if self.dist_on:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, x: float) -> float:
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        if self.dist_on:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def events(self, n):
        E = self.torch.cuda.Event
        return [(E(enable_timing=True), E(enable_timing=True)) for _ in range(n)]

    def timed(self, fn, steps, warmup, kern=None):
        """fn() enqueues one bench step on self.stream; kern (optional) is a list that fn fills with
        (start, end) events around the dominant kernel's launches.  Returns (per-step ms list,
        per-step kernel ms list)."""
        for _ in range(warmup):
            with self.torch.cuda.stream(self.stream):
                fn(None)
        self.barrier()
        ev = self.events(steps)
        kev = self.events(steps)
        for i in range(steps):
            self.flush()  # untimed L2 flush between iterations
            ev[i][0].record(self.stream)
            with self.torch.cuda.stream(self.stream):
                fn(kev[i])
            ev[i][1].record(self.stream)
        self.barrier()
        return [s.elapsed_time(e) for s, e in ev], [s.elapsed_time(e) for s, e in kev]


def hbm_roofline(alg_bytes_per_launch, kern_s, kernel, traffic=None, note=None):
    peak, src = measured_peak()
    ach = alg_bytes_per_launch / kern_s / 1e9
    d = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
         "traffic": traffic, "peak_source": src, "kernel": kernel, "alg_bytes_per_launch": alg_bytes_per_launch,
         "kernel_ms": kern_s * 1e3}
    if traffic:
        d["dram_GBps"] = traffic / kern_s / 1e9
        d["dram_frac"] = d["dram_GBps"] / peak
    if note:
        d["note"] = note
    return d


def issue_roofline(kernel, kern_s, clocks, inst=None, traffic=None, hbm=None, counters_source=None):
    """Issue-bound roofline: ncu smsp__inst_executed per launch (or run) / kernel time against
    148 SMs x 4 SMSPs x 1 warp-instruction per cycle at the median SM clock under load; the HBM
    figures ride along in "hbm" (actual DRAM traffic from the same capture)."""
    sm_ghz = (clocks.get("sm_mhz") or 1965.0) / 1e3
    peak = 148 * 4 * sm_ghz  # warp-instructions per ns
    hbm_peak, hbm_src = measured_peak()
    roof = {"bound": "issue", "kernel": kernel, "kernel_ms": kern_s * 1e3, "unit": "G warp-inst/s", "peak": peak,
            "peak_source": f"148 SMs x 4 SMSPs x 1 warp-inst/cycle x {sm_ghz:.3f} GHz (median SM clock under load)",
            "achieved": None, "frac": None, "traffic": traffic,
            "hbm": dict(hbm or {}, peak=hbm_peak, peak_source=hbm_src)}
    if inst:
        roof["achieved"] = inst / kern_s / 1e9
        roof["frac"] = roof["achieved"] / peak
        roof["inst_executed"] = inst
        roof["counters_source"] = counters_source
    if traffic:
        roof["hbm"]["dram_GBps"] = traffic / kern_s / 1e9
        roof["hbm"]["dram_frac"] = roof["hbm"]["dram_GBps"] / hbm_peak
    return roof


def bench_c1(cx: Ctx, clk):
    import paper_2512_06102_b200 as eb
    torch = cx.torch
    a, s = cx.args, SPEC["C1"]
    env0, n = rank_envs("C1", cx.rank, cx.world, a.scaling)
    h, w, steps = s["h"], s["w"], s["steps"]
    terrain = eb.synth_terrain(SEED, n, h, w, env_id0=env0)
    init = eb.synth_ignitions(SEED, terrain, s["ignitions"], env_id0=env0)
    b = eb.Batch(n, h, w, device=cx.local, stream=cx.stream.cuda_stream)
    b.set_terrain(terrain.fuel_class, terrain.elevation, terrain.class_veg, terrain.class_den, 30.0)
    b.set_wind(terrain.wind_speed, terrain.wind_direction)
    b.set_config(None)
    b.set_kernel({"auto": 0, "tiled": 1, "resident": 2, "warp": 6}[a.kernel])
    b.set_key(SEED, 0, first_stream=env0)
    init_dev = torch.from_numpy(init).to(cx.dev)
    L = eb.lib()

    def step(kev):
        eb._lib.check(L.ebl_batch_set_state_device(b.handle, init_dev.data_ptr()))
        b.set_key(SEED, 0, first_stream=env0)
        if kev:
            kev[0].record(cx.stream)
        b.step(steps)
        if kev:
            kev[1].record(cx.stream)

    b.diag(reset=True)
    clk.__enter__()
    ms, kms = cx.timed(step, a.steps, a.warmup)
    diag = b.diag()
    units = n * h * w * steps
    t_max = cx.max_over_ranks(sum(ms) / 1e3)
    total_units = cx.sum_over_ranks(units * a.steps)
    value = total_units / t_max

    # ---- end to end: the public host-buffer call (copy in, 200 fused steps, copy out) ----------
    h_in = eb.host_buffer(init.shape)
    h_in[:] = init
    h_out = eb.host_buffer(init.shape)
    eb._lib.check(L.ebl_batch_set_pipeline(b.handle, a.pipeline))

    def e2e_step():
        eb._lib.check(L.ebl_batch_set_key(b.handle, SEED, 0, None, env0))
        eb._lib.check(L.ebl_batch_run(b.handle, h_in.ctypes.data, steps, h_out.ctypes.data))

    for _ in range(2):
        e2e_step()
    cx.barrier()
    e2e_ms = []
    for _ in range(a.steps):
        cx.flush()
        cx.barrier()
        e0, e1 = cx.events(1)[0]
        e0.record(cx.stream)
        e2e_step()
        e1.record(cx.stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    clk.__exit__(None, None, None)
    te = cx.max_over_ranks(sum(e2e_ms) / 1e3)
    e2e_value = total_units / te
    final_dev = b.get_state()
    assert np.array_equal(h_out, final_dev), "e2e result differs from the device run"

    kern_s = sum(kms) / len(kms) / 1e3
    alg = units * ALG_BYTES["C1"]
    cnt = ncu_counters(f"k_step_warp:{n}x{h}x{w}x{steps}") or {}
    hbm_peak, _ = measured_peak()
    roof = issue_roofline("k_step_warp", kern_s, clk.summary(), inst=cnt.get("inst_executed_per_launch"),
                          traffic=cnt.get("dram_bytes_per_launch"), counters_source=cnt.get("source"),
                          hbm={"alg_bytes_per_launch": alg, "alg_GBps": alg / kern_s / 1e9,
                               "alg_frac": alg / kern_s / 1e9 / hbm_peak,
                               "note": "SURVEY §8(d) 10 B/cell-update; exceeds 1 because the state stays in "
                                       "shared memory for all 200 steps (DRAM sees the layers once per run)"})
    res = dict(value=value, ms_per_step=t_max * 1e3 / a.steps, units_per_rank=units,
               e2e={"value": e2e_value, "unit": s["unit"], "h2d_bytes_per_step": int(init.nbytes),
                    "d2h_bytes_per_step": int(init.nbytes), "ms_per_step": te * 1e3 / a.steps},
               roofline=roof, gpu_launches=diag["launches"],
               extra={"env_steps_per_sec": value / (h * w), "fp64_fallback_draws": diag["fp64_fallbacks"],
                      "ambiguous_draws": diag["ambiguous"]})
    b.close()
    return res


def bench_c0(cx: Ctx, clk):
    import paper_2512_06102_b200 as eb
    torch = cx.torch
    a = cx.args
    h = w = 64
    z = np.zeros((h, w))
    b = eb.Batch(1, h, w, device=cx.local, stream=cx.stream.cuda_stream)
    b.set_grid(z, z, z, z, np.zeros((h, w, 8)))
    fire = np.zeros((1, h, w), np.uint8)
    fire[0, 32, 32] = 1
    dev = torch.from_numpy(fire).to(cx.dev)
    L = eb.lib()

    def step(kev):
        eb._lib.check(L.ebl_batch_set_state_device(b.handle, dev.data_ptr()))
        b.set_key(0, 0)
        if kev:
            kev[0].record(cx.stream)
        b.step(100)
        if kev:
            kev[1].record(cx.stream)
    b.diag(reset=True)
    clk.__enter__()
    ms, kms = cx.timed(step, a.steps, a.warmup)
    diag = b.diag()
    units = h * w * 100
    t_max = cx.max_over_ranks(sum(ms) / 1e3)
    value = cx.sum_over_ranks(units * a.steps) / t_max
    # e2e: the one-shot run_stochastic signature (host buffers, general-form tables built inside)
    grid = dict(speed=z, dir=z, veg=z, den=z, slope8=np.zeros((h, w, 8)))
    eb.run_stochastic(fire[0], grid, None, (0, 0, 0), 100)
    cx.barrier()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        out = eb.run_stochastic(fire[0], grid, None, (0, 0, 0), 100)
    e2e_s = cx.max_over_ranks(time.perf_counter() - t0)
    clk.__exit__(None, None, None)
    assert np.array_equal(out, b.get_state()[0])
    kern_s = sum(kms) / len(kms) / 1e3
    return dict(value=value, ms_per_step=t_max * 1e3 / a.steps, units_per_rank=units,
                e2e={"value": units * a.steps / e2e_s, "unit": SPEC["C0"]["unit"],
                     "h2d_bytes_per_step": int(fire.nbytes + 5 * z.nbytes + 8 * z.nbytes),
                     "d2h_bytes_per_step": int(fire.nbytes), "note": "host-timed ebl_run_stochastic"},
                roofline=hbm_roofline(units * 10, kern_s, "k_step_warp",
                                      note="latency-bound: one 100-step launch of a 4096-cell env (1 CTA)"),
                gpu_launches=diag["launches"], extra={})


def bench_c2(cx: Ctx, clk):
    import paper_2512_06102_b200 as eb
    torch = cx.torch
    a, s = cx.args, SPEC["C2"]
    env0, n = rank_envs("C2", cx.rank, cx.world, a.scaling)
    h, w, steps = s["h"], s["w"], s["steps"]
    t = eb.synth_terrain(SEED, n, h, w, env_id0=env0)
    env = eb.VecFireEnv(n, variant=eb.RL_TANKER, terrain=t, sim_cfg=None, ignitions=s["ignitions"],
                        max_steps=256, env_id0=env0, device=cx.local, stream=cx.stream.cuda_stream)
    env.reset(SEED)
    L = eb.lib()
    hnd = env.batch.handle

    def step(kev):
        if kev:
            kev[0].record(cx.stream)
        eb._lib.check(L.ebl_rl_rollout(hnd, steps, None, None))
        if kev:
            kev[1].record(cx.stream)
    env.batch.diag(reset=True)
    clk.__enter__()
    ms, kms = cx.timed(step, a.steps, a.warmup)
    launches = env.batch.diag()["launches"]
    units = n * steps
    t_max = cx.max_over_ranks(sum(ms) / 1e3)
    total = cx.sum_over_ranks(units * a.steps)
    value = total / t_max
    # e2e: the per-step C-ABI call with host actions in and host reward/done out, every step
    act = eb.host_buffer((steps, n), np.int32)
    rs = np.random.default_rng(1)
    act[:] = rs.integers(0, h * w, (steps, n), dtype=np.int32)
    rew = eb.host_buffer((n,), np.float64)
    done = eb.host_buffer((n,), np.uint8)

    def e2e_step():
        for k in range(steps):
            eb._lib.check(L.ebl_rl_step(hnd, act[k].ctypes.data, rew.ctypes.data, done.ctypes.data, 0))
    e2e_step()
    cx.barrier()
    e2e_ms = []
    for _ in range(a.steps):
        cx.flush()
        cx.barrier()
        e0, e1 = cx.events(1)[0]
        e0.record(cx.stream)
        e2e_step()
        e1.record(cx.stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    # learner in the loop: device actions/reward/done (ebl_rl_step device_io=1), no host round trip
    dact = torch.from_numpy(np.ascontiguousarray(act)).to(cx.dev)
    drew = torch.empty(n, dtype=torch.float64, device=cx.dev)
    ddone = torch.empty(n, dtype=torch.uint8, device=cx.dev)

    def dev_step(kev):
        if kev:
            kev[0].record(cx.stream)
        for k in range(steps):
            eb._lib.check(L.ebl_rl_step(hnd, dact[k].data_ptr(), drew.data_ptr(), ddone.data_ptr(), 1))
        if kev:
            kev[1].record(cx.stream)
    dms, _ = cx.timed(dev_step, max(2, a.steps // 2), 1)
    clk.__exit__(None, None, None)
    te = cx.max_over_ranks(sum(e2e_ms) / 1e3)
    kern_s = sum(kms) / len(kms) / 1e3
    cnt = ncu_counters(f"k_rl_tanker_warp:{n}x{h}x{w}x{steps}")
    return dict(value=value, ms_per_step=t_max * 1e3 / a.steps, units_per_rank=units,
                e2e={"value": total / te, "unit": s["unit"], "h2d_bytes_per_step": int(act.nbytes),
                     "d2h_bytes_per_step": int(steps * (rew.nbytes + done.nbytes)),
                     "note": "ebl_rl_step per RL step: host actions in, host reward/done out"},
                roofline=issue_roofline(
                    "k_rl_tanker_warp", kern_s, clk.summary(), inst=(cnt or {}).get("inst_executed_per_launch"),
                    traffic=(cnt or {}).get("dram_bytes_per_launch"), counters_source=(cnt or {}).get("source"),
                    hbm={"alg_bytes_per_launch": units * ALG_BYTES["C2"],
                         "alg_GBps": units * ALG_BYTES["C2"] / kern_s / 1e9,
                         "note": "one fused 256-step launch; the layers stay in shared memory (bit planes), "
                                 "so the algorithmic bytes exceed the DRAM traffic"}),
                gpu_launches=launches,
                extra={"cell_updates_per_sec": value * h * w,
                       "device_io_step": {"env_steps_per_sec": cx.sum_over_ranks(units * len(dms))
                                          / cx.max_over_ranks(sum(dms) / 1e3),
                                          "note": "ebl_rl_step(device_io=1) per RL step with device "
                                                  "actions/reward/done (learner in the loop)"}})


def bench_c3(cx: Ctx, clk):
    import paper_2512_06102_b200 as eb
    from paper_2512_06102_b200 import sharded as SH
    torch = cx.torch
    a, s = cx.args, SPEC["C3"]
    H, W, steps, K = s["h"], s["w"], s["steps"], 16  # the tiles' light-cone halo (kBlockHalo)
    shards = SH.plan_shards(H, cx.world, K)
    me = shards[cx.rank]
    g0, g1 = me.rows
    b = eb.Batch(1, g1 - g0, W, device=cx.local, stream=cx.stream.cuda_stream)
    # environment construction on the device (the C1 generator, bit-identical to the host one)
    full = eb.Batch(1, H, W, device=cx.local, stream=cx.stream.cuda_stream) if cx.world > 1 else b
    full.synth_terrain(SEED)
    full.set_wind([6.0], [0.0])
    full.synth_ignitions(SEED, s["ignitions"])
    L = eb.lib()
    if cx.world > 1:
        fc, el = full.get_terrain()
        init = full.get_state()
        full.close()
        _, veg, den = eb.worldcover_palette()
        b.set_terrain(fc[:, g0:g1], el[:, g0:g1], veg, den, 30.0)
        b.set_wind([6.0], [0.0])
        eb._lib.check(L.ebl_batch_set_row_offset(b.handle, g0))
        eb._lib.check(L.ebl_batch_set_band(b.handle, me.band[0] - g0, me.band[1] - g0))
        init = init[:, g0:g1]
        del fc, el
    else:
        init = b.get_state()
    b.set_config(None)
    init_dev = torch.from_numpy(np.ascontiguousarray(init)).to(cx.dev)
    rows_buf = {}

    def get_rows(r0, n):
        t = torch.empty((n, W), dtype=torch.uint8, device=cx.dev)
        eb._lib.check(L.ebl_batch_rows_device(b.handle, r0, n, t.data_ptr(), 0))
        return t

    def set_rows(r0, t):
        eb._lib.check(L.ebl_batch_rows_device(b.handle, r0, t.shape[0], t.data_ptr(), 1))

    def make_buffer(n):
        return rows_buf.setdefault(n, torch.empty((n, W), dtype=torch.uint8, device=cx.dev))

    def run_steps():
        if cx.world == 1:
            b.step(steps)
        else:
            done = 0
            while done < steps:
                k = min(K, steps - done)
                b.step(k)
                SH.exchange_halos(cx.dist, cx.rank, shards, get_rows, set_rows, make_buffer)
                done += k

    def step(kev):
        eb._lib.check(L.ebl_batch_set_state_device(b.handle, init_dev.data_ptr()))
        b.set_key(SEED, 0)
        if kev:
            kev[0].record(cx.stream)
        run_steps()
        if kev:
            kev[1].record(cx.stream)
    b.diag(reset=True)
    clk.__enter__()
    ms, kms = cx.timed(step, a.steps, max(1, a.warmup - 2))
    diag = b.diag()
    units = H * W * steps
    t_max = cx.max_over_ranks(sum(ms) / 1e3)
    value = units * a.steps / t_max
    kern_s = sum(kms) / len(kms) / 1e3

    # ---- end to end: the landscape (this rank's rows) from pinned host memory, 500 steps, back ----
    h_in = eb.host_buffer(init.shape)
    h_in[:] = init
    h_out = eb.host_buffer(init.shape)

    def e2e_step():
        eb._lib.check(L.ebl_batch_set_state(b.handle, h_in.ctypes.data))
        b.set_key(SEED, 0)
        run_steps()
        eb._lib.check(L.ebl_batch_get_state(b.handle, h_out.ctypes.data))

    e2e_step()
    cx.barrier()
    e2e_ms = []
    for _ in range(a.steps):
        cx.flush()
        cx.barrier()
        e0, e1 = cx.events(1)[0]
        e0.record(cx.stream)
        e2e_step()
        e1.record(cx.stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    clk.__exit__(None, None, None)
    assert np.array_equal(h_out, b.get_state()), "e2e result differs from the device run"
    te = cx.max_over_ranks(sum(e2e_ms) / 1e3)
    tiles = diag.get("tiles_processed"), diag.get("tiles_launched")
    active = None
    if tiles[0] is not None and tiles[1]:
        active = value * tiles[0] / tiles[1]
    # issue-bound roofline over one run's launches (the active tiles' 8-step chains), HBM beside it
    cnt = (ncu_counters(f"k_step_warp:c3:{H}x{W}x{steps}") if cx.world == 1 else None) or {}
    roof = issue_roofline("k_step_warp (halo tiles, work lists; per run of 500 steps)", kern_s, clk.summary(),
                          inst=cnt.get("inst_executed_per_run"), traffic=cnt.get("dram_bytes_per_run"),
                          counters_source=cnt.get("source"),
                          hbm={"note": "SURVEY §8(d) counts 10 B per dense cell-update; only the active tiles "
                                       "are read and written (tiles_processed_frac)"})
    return dict(value=value, ms_per_step=t_max * 1e3 / a.steps, units_per_rank=units // cx.world,
                e2e={"value": units * a.steps / te, "unit": s["unit"], "h2d_bytes_per_step": int(init.nbytes),
                     "d2h_bytes_per_step": int(init.nbytes), "ms_per_step": te * 1e3 / a.steps},
                roofline=roof, gpu_launches=diag["launches"],
                extra={"launches_per_run": diag["launches"] // max(1, a.steps + max(1, a.warmup - 2)),
                       "tiles_processed_frac": (tiles[0] / tiles[1]) if active else None,
                       "active_tile_cell_updates_per_sec": active})


def bench_c4(cx: Ctx, clk):
    import paper_2512_06102_b200 as eb
    torch = cx.torch
    a, s = cx.args, SPEC["C4"]
    env0, n = rank_envs("C4", cx.rank, cx.world, a.scaling)
    h, w, steps = s["h"], s["w"], s["steps"]
    t = eb.synth_terrain(4, n, h, w, env_id0=env0)
    init = eb.synth_ignitions(4, t, s["ignitions"], env_id0=env0)
    b = eb.Batch(n, h, w, device=cx.local, stream=cx.stream.cuda_stream)
    b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed, t.wind_direction)
    b.set_config(None)
    mask = (np.random.default_rng(env0).random((n, h, w)) < 0.2).astype(np.float64)
    b.set_state(init)
    b.det_set_state_from_fire()
    b.det_forward(1, record=True)   # builds the tables once (setup)
    b.det_set_mask(mask)            # the calibration target, resident (as ebl_calibrate keeps it)
    init_dev = torch.from_numpy(init).to(cx.dev)
    L = eb.lib()
    loss = np.empty(n)
    grad = np.empty((n, 6))

    def step(kev):
        eb._lib.check(L.ebl_batch_set_state_device(b.handle, init_dev.data_ptr()))
        if kev:
            kev[0].record(cx.stream)
        eb._lib.check(L.ebl_det_set_state_from_fire(b.handle))
        eb._lib.check(L.ebl_det_forward(b.handle, steps, 1))
        eb._lib.check(L.ebl_det_loss_grad(b.handle, None, 0.0, 1.0, 1, loss.ctypes.data, grad.ctypes.data))
        if kev:
            kev[1].record(cx.stream)
    b.diag(reset=True)
    clk.__enter__()
    ms, kms = cx.timed(step, a.steps, a.warmup)
    launches = b.diag()["launches"]
    units = n * h * w * steps
    t_max = cx.max_over_ranks(sum(ms) / 1e3)
    total = cx.sum_over_ranks(units * a.steps)
    value = total / t_max
    # e2e: host fire layers in (state_from_fire on the device), host target mask in, host loss and
    # gradient out, every step
    h_init = eb.host_buffer(init.shape)
    h_init[:] = init
    h_mask = eb.host_buffer(mask.shape, np.float64)
    h_mask[:] = mask

    def e2e_step():
        eb._lib.check(L.ebl_batch_set_state(b.handle, h_init.ctypes.data))
        eb._lib.check(L.ebl_det_set_state_from_fire(b.handle))
        eb._lib.check(L.ebl_det_forward(b.handle, steps, 1))
        eb._lib.check(L.ebl_det_loss_grad(b.handle, h_mask.ctypes.data, 0.0, 1.0, 1, loss.ctypes.data,
                                          grad.ctypes.data))
    e2e_step()
    cx.barrier()
    e2e_ms = []
    for _ in range(a.steps):
        cx.flush()
        cx.barrier()
        e0, e1 = cx.events(1)[0]
        e0.record(cx.stream)
        e2e_step()
        e1.record(cx.stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    clk.__exit__(None, None, None)
    te = cx.max_over_ranks(sum(e2e_ms) / 1e3)
    kern_s = sum(kms) / len(kms) / 1e3
    cnt = ncu_counters(f"c4:{n}x{h}x{w}x{steps}")
    # the calibration loop at this size (calibrate.cpp:104-167): each iteration sets theta, builds
    # the SpreadTables on the device, runs the recorded rollout, the loss and the gradient, Adam on
    # the 6 parameters; per-iteration cost = (T(4 iterations) - T(0)) / 4, host-timed (both run
    # iteration 0's rollout; the difference is four more iterations)
    planes = [(init == k).astype(np.float64) for k in (0, 1, 2)]
    cal_t = {}
    for iters in (0, 4, 0, 4):
        cx.barrier()
        t0 = time.perf_counter()
        b.calibrate(*planes, mask, steps, iterations=iters, bce_weight=0.0, mse_weight=1.0, pool=1)
        cal_t[iters] = time.perf_counter() - t0  # the second of each pair: warm
    cal_ms = (cal_t[4] - cal_t[0]) / 4 * 1e3
    return dict(value=value, ms_per_step=t_max * 1e3 / a.steps, units_per_rank=units,
                e2e={"value": total / te, "unit": s["unit"], "h2d_bytes_per_step": int(init.nbytes + mask.nbytes),
                     "d2h_bytes_per_step": int(loss.nbytes + grad.nbytes)},
                roofline=hbm_roofline(units * ALG_BYTES["C4"], kern_s, "k_det_forward + k_det_back (per step)",
                                      traffic=cnt.get("dram_bytes_per_run") if cnt else None,
                                      note="fp64 forward (100 launches) + loss + fused backward (100 launches)"),
                gpu_launches=launches, extra={"loss_sum": float(loss.sum()),
                                              "calibrate_ms_per_iteration": cal_ms,
                                              "calibrate_s": {"iterations_0": cal_t[0], "iterations_4": cal_t[4]},
                                              "calibrate_note": "ebl_calibrate at C4 size: tables built on the "
                                                                "device each iteration (no host table build)"})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C1", choices=sorted(SPEC))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "tiled", "resident", "warp"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pipeline", type=int, default=0,
                    help="env chunks of the C1 e2e host-buffer pipeline (0 = library default)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.config in ("C0", "C3"):
        args.scaling = "strong" if args.config == "C3" else args.scaling

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    cx = Ctx(args, rank, world, local)
    clk = ClockSampler(local)
    fn = {"C0": bench_c0, "C1": bench_c1, "C2": bench_c2, "C3": bench_c3, "C4": bench_c4}[args.config]
    res = fn(cx, clk)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_sample(args.config, {"C0": 3.0, "C1": 15.0, "C2": 10.0, "C3": 15.0, "C4": 15.0}[args.config])
        cpu = {"value": r["units"] / r["seconds"], "unit": SPEC[args.config]["unit"], "cores": r["cores"],
               "kind": r["kind"], "sample": r["sample"] + f" ({r['units']:.3g} units, {r['seconds']:.1f} s)"}
    if rank == 0:
        s = SPEC[args.config]
        line = {"metric": s["metric"], "value": res["value"], "unit": s["unit"], "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": "u8+f32" if args.config != "C4" else "f64",
                "data": "synthetic (seeded generator, DESIGN.md §5)",
                "config": config_json(args.config, world, args.scaling), "impl": "ours",
                "e2e": res["e2e"], "roofline": res["roofline"], "gpu_launches": res["gpu_launches"],
                "clocks": clk.summary(), "cpu_baseline": cpu}
        line.update(res["extra"])
        print(json.dumps(line), flush=True)
    if cx.dist_on:
        cx.dist.barrier()
        cx.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
