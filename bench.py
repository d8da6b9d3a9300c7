"""Benchmark of the batched CA fire-spread step (BASELINE.json metric, config C1).

Workload (configs[1]): 1024 independent envs of 128x128, per-env seeded landcover/elevation/
wind, 5 ignitions per env, 200 CA steps.  One bench "step" = one full C1 run on the GPU:
reset the 1024 fire layers to their ignitions and advance 200 CA steps
(= 1024*16384*200 = 3.36e9 cell-updates, counted densely as emberline_main.cpp:432-433).

  value   device throughput, inputs resident in HBM, CUDA events on the launch stream,
          L2 flushed (256 MiB write) between timed iterations, max over ranks.
  e2e     the same metric through the public C-ABI with HOST buffers (ebl_batch_run):
          pinned host -> device copy of the 1024 initial layers, 200 steps, device -> host
          copy of the 1024 final layers, all inside the timed region; the library pipelines
          the copies against the compute over env chunks.
  roofline  dominant kernel (k_step_blocked) vs measured HBM copy bandwidth, at SURVEY
          §8(d)'s 10 algorithmic bytes per cell-update.
  cpu_baseline  the reference's own code (oracle/_ref = /root/reference/proj compiled in
          place) on this host's cores, a bounded sample of the same workload.

Multi-GPU (torchrun): one process per GPU, envs sharded by global env id (weak scaling:
each rank runs its own 1024 envs, ids rank*1024..), no data-path collective.
`--impl reference` runs only the reference CPU arm (rank 0), same metric/config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ENVS, H, W, CA_STEPS, IGNITIONS, SEED = 1024, 128, 128, 200, 5, 0
ALG_BYTES_PER_CELL_UPDATE = 10  # 1 B state read + 1 B write + 4 B fuel + 4 B elevation


def config_json(world: int, kernel: str) -> dict:
    """The workload description shared by both arms (BASELINE.json configs[1])."""
    return {"workload": "C1: 1024 envs x 128x128 per GPU, per-env value-noise landcover "
                        "(11 WorldCover classes) + fractal elevation 0-500 m + wind "
                        "U(0,10)/U(0,2pi), 5 ignitions, 200 CA steps",
            "global_batch": N_ENVS * world, "grid": [H, W], "ca_steps": CA_STEPS,
            "parallelism": f"env-sharded x{world}", "kernel": kernel,
            "l2": "flushed between timed iterations (256 MiB write)"}


def env_ids(rank: int) -> list:
    """Global env ids (= RNG streams, = synthetic-terrain keys) of a rank: weak scaling,
    each rank owns its own N_ENVS envs; no data-path collective."""
    return list(range(rank * N_ENVS, (rank + 1) * N_ENVS))


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


def cpu_reference_sample(n_envs: int, threads: int = 0):
    """Times the reference (or, without it, the C port) on n_envs C1 envs x 200 steps.
    Returns (seconds, cell_updates, kind, cores, digest_ok)."""
    from oracle import oracle as O
    import paper_2512_06102_b200 as eb
    t = eb.synth_terrain(SEED, n_envs, H, W)
    init = eb.synth_ignitions(SEED, t, IGNITIONS)
    cfg = O.cfg_array(O.DEFAULT_CFG)
    streams = np.arange(n_envs, dtype=np.uint64)
    R = O.ref()
    kind = "reference" if R is not None else "port"
    L = R if R is not None else O.port()
    grids = [(O.grid_terrain(L, "ref" if R is not None else "port", t.veg()[e], t.den()[e],
                             t.elevation[e], 30.0, t.wind_speed[e], t.wind_direction[e]))
             for e in range(n_envs)]
    handles = (O._P * n_envs)(*[g.h for g in grids])
    states = np.ascontiguousarray(init.copy())
    fn = L.ref_run_envs if R is not None else L.ebo_run_envs
    secs = fn(handles, n_envs, O.ptr(cfg), SEED, O.ptr(streams), CA_STEPS, O.ptr(states), threads)
    cores = (R.ref_max_threads() if R is not None else os.cpu_count()) if threads <= 0 else threads
    return secs, n_envs * H * W * CA_STEPS, kind, cores, states


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    cfgj = config_json(world, "reference CPU (emberline run_stochastic)")
    # each bench step = a bounded sample of the workload, sized to ~2-4 s of CPU work
    secs, cells, kind, cores, _ = cpu_reference_sample(4)
    n_sample = int(max(4, min(N_ENVS, 4 * 3.0 / max(secs, 1e-3))))
    for _ in range(args.warmup):
        cpu_reference_sample(n_sample)
    times, tot_cells = [], 0
    for _ in range(args.steps):
        s, c, kind, cores, _ = cpu_reference_sample(n_sample)
        times.append(s)
        tot_cells += c
    value = tot_cells / sum(times)
    line = {"metric": "cell-updates/sec", "value": value, "unit": "cell-updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfgj, "impl": "reference",
            "env_steps_per_sec": value / (H * W),
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": kind,
                             "sample": f"{n_sample} of the 1024 C1 envs x 200 steps per bench step "
                                       "(run_stochastic per env, Exec::serial, OpenMP over envs)"},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "tiled", "resident", "paired", "frontier", "warp", "warp2"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pipeline", type=int, default=0,
                    help="env chunks of the e2e host-buffer pipeline (0 = library default)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2512_06102_b200 as eb

    dist_on = world > 1
    torch.cuda.set_device(local)
    if dist_on:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    env0 = env_ids(rank)[0]  # global env ids of this rank (weak scaling)
    terrain = eb.synth_terrain(SEED, N_ENVS, H, W, env_id0=env0)
    init = eb.synth_ignitions(SEED, terrain, IGNITIONS, env_id0=env0)

    stream = torch.cuda.Stream()
    b = eb.Batch(N_ENVS, H, W, device=local, stream=stream.cuda_stream)
    b.set_terrain(terrain.fuel_class, terrain.elevation, terrain.class_veg, terrain.class_den, 30.0)
    b.set_wind(terrain.wind_speed, terrain.wind_direction)
    b.set_config(None)
    b.set_kernel({"auto": 0, "tiled": 1, "resident": 2, "paired": 4, "frontier": 5, "warp": 6, "warp2": 7}[args.kernel])
    b.set_key(SEED, 0, first_stream=env0)

    init_dev = torch.from_numpy(init).to(f"cuda:{local}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2

    def device_step():
        eb._lib.check(eb.lib().ebl_batch_set_state_device(b.handle, init_dev.data_ptr()))
        b.set_key(SEED, 0, first_stream=env0)
        b.step(CA_STEPS)

    def barrier():
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()

    # ---- device-resident throughput -------------------------------------------------------
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            device_step()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kern_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    b.diag(reset=True)
    clk = ClockSampler(local).__enter__()   # sampled over both timed regions (device and e2e)
    barrier()
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()                       # untimed L2 flush between iterations
            ev[i][0].record(stream)
            eb._lib.check(eb.lib().ebl_batch_set_state_device(b.handle, init_dev.data_ptr()))
            b.set_key(SEED, 0, first_stream=env0)
            kern_ev[i][0].record(stream)
            b.step(CA_STEPS)
            kern_ev[i][1].record(stream)
            ev[i][1].record(stream)
    barrier()
    diag = b.diag()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    kern_ms = [s.elapsed_time(e) for s, e in kern_ev]
    t_local = sum(step_ms) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device=f"cuda:{local}")
    if dist_on:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    cells_per_rank = N_ENVS * H * W * CA_STEPS * args.steps
    value = cells_per_rank * world / t_max

    # ---- end to end through the C-ABI with host buffers ---------------------------------------
    # host buffers: pinned, mapped, huge-page memory from the library's allocator (ebl_host_alloc)
    h_in = eb.host_buffer(init.shape)
    h_in[:] = init
    h_out = eb.host_buffer(init.shape)
    L = eb.lib()
    in_ptr, out_ptr = h_in.ctypes.data, h_out.ctypes.data

    eb._lib.check(L.ebl_batch_set_pipeline(b.handle, args.pipeline))

    def e2e_step():  # the public host-buffer call: copy in, 200 fused steps, copy out (pipelined)
        eb._lib.check(L.ebl_batch_set_key(b.handle, SEED, 0, None, env0))
        eb._lib.check(L.ebl_batch_run(b.handle, in_ptr, CA_STEPS, out_ptr))

    for _ in range(2):
        e2e_step()
    barrier()
    e2e_ms = []
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    clk.__exit__(None, None, None)
    te = torch.tensor([sum(e2e_ms) / 1e3], dtype=torch.float64, device=f"cuda:{local}")
    if dist_on:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = cells_per_rank * world / float(te.item())
    # result check against the device run (same key => same final layers)
    final_dev = b.get_state()
    assert np.array_equal(h_out, final_dev), "e2e result differs from the device run"

    # ---- roofline of the dominant kernel --------------------------------------------------------
    peak, peak_src = measured_peak()
    kern_s = sum(kern_ms) / len(kern_ms) / 1e3
    alg_bytes = N_ENVS * H * W * CA_STEPS * ALG_BYTES_PER_CELL_UPDATE
    achieved = alg_bytes / kern_s / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("kernel_config") == f"{args.kernel}:{N_ENVS}x{H}x{W}x{CA_STEPS}":
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        secs, cells, kind, cores, _ = cpu_reference_sample(4)
        n_sample = int(max(4, min(N_ENVS, 4 * 15.0 / max(secs, 1e-3))))
        secs, cells, kind, cores, _ = cpu_reference_sample(n_sample)
        cpu = {"value": cells / secs, "unit": "cell-updates/s", "cores": cores, "kind": kind,
               "sample": f"{n_sample} of the 1024 C1 envs x 200 steps ({cells:.3g} cell-updates, "
                         f"{secs:.1f} s; run_stochastic per env, Exec::serial, OpenMP over envs)"}

    if rank == 0:
        line = {
            "metric": "cell-updates/sec", "value": value, "unit": "cell-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": config_json(world, args.kernel),
            "env_steps_per_sec": value / (H * W),
            "e2e": {"value": e2e_value, "unit": "cell-updates/s",
                    "h2d_bytes_per_step": int(init.nbytes), "d2h_bytes_per_step": int(init.nbytes)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": {"tiled": "k_step_tile", "frontier": "k_step_frontier", "resident": "k_step_blocked",
                                    "paired": "k_step_blocked", "warp2": "k_step_warp2"}.get(
                             args.kernel, "k_step_warp"),
                         "alg_bytes_per_launch": alg_bytes if args.kernel != "tiled"
                         else alg_bytes // CA_STEPS,
                         "kernel_ms": kern_s * 1e3},
            "gpu_launches": diag["launches"],
            "fp64_fallback_draws": diag["fp64_fallbacks"], "ambiguous_draws": diag["ambiguous"],
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()
    b.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
