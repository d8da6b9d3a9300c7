"""Python mirror of the reference's engine / RL interface on top of the C-ABI.

Names and argument meaning follow proj/include/emberline/engine.hpp and
rl_env.hpp (cited per method) so the parity tests read like the reference's own
tests.  Arrays are numpy; state layers are uint8 [..., H, W] with row 0 = south.
Everything runs on the GPU through libember_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import EnvConfig, EnvState, SimConfig, check, lib

UNBURNED, BURNING, BURNED = 0, 1, 2
KERNEL_AUTO, KERNEL_TILED, KERNEL_RESIDENT, KERNEL_BLOCKED, KERNEL_WARP = 0, 1, 2, 3, 6


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


class _HostMem:
    """Owner of an ebl_host_alloc block (freed with the last array viewing it)."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        check(lib().ebl_host_alloc(nbytes, C.byref(p)))
        self.ptr, self.nbytes = p.value, nbytes
        self.buf = (C.c_char * nbytes).from_address(self.ptr)

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().ebl_host_free(C.c_void_p(self.ptr))
            self.ptr = None


def host_buffer(shape, dtype=np.uint8) -> np.ndarray:
    """A numpy array in pinned, mapped, huge-page host memory (ebl_host_alloc): the host buffers
    to hand Batch.run / set_state / get_state for full-rate transfers."""
    shape = (shape,) if isinstance(shape, int) else tuple(shape)
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    mem = _HostMem(max(nbytes, 1))
    arr = np.frombuffer(mem.buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    mem.buf._owner = mem  # the ctypes buffer (the arrays' base) keeps the allocation alive
    return arr


def parse_snapshot(text: str | bytes):
    """parse_snapshot (snapshot.cpp:74-121): (layer [H, W] uint8, step, agent (row, col, water) or
    None); malformed text raises FileError with the reference's message."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    h, w, step, ha = C.c_int(), C.c_int(), C.c_uint64(), C.c_int()
    check(lib().ebl_snapshot_parse(b, len(b), C.byref(h), C.byref(w), C.byref(step), None, 0, None, C.byref(ha)))
    layer = np.empty((h.value, w.value), np.uint8)
    ag = np.zeros(3, np.int32)
    check(lib().ebl_snapshot_parse(b, len(b), C.byref(h), C.byref(w), C.byref(step), _ptr(layer), layer.size,
                                   _ptr(ag), C.byref(ha)))
    return layer, step.value, (tuple(int(x) for x in ag) if ha.value else None)


def default_config(**overrides) -> SimConfig:
    """SimConfig{} (grid.hpp:173-179) with keyword overrides."""
    c = SimConfig()
    lib().ebl_default_config(C.byref(c))
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def as_config(cfg) -> SimConfig:
    if cfg is None:
        return default_config()
    if isinstance(cfg, SimConfig):
        return cfg
    if isinstance(cfg, dict):
        return default_config(**cfg)
    vals = list(cfg)
    return default_config(p_base=vals[0], alpha_w1=vals[1], alpha_w2=vals[2], alpha_s=vals[3],
                          alpha_gamma=vals[4], p_continue=vals[5])


def validate_config(cfg) -> None:
    """validate_config (grid.cpp:107-124): raises InvalidArgument."""
    check(lib().ebl_validate_config(C.byref(as_config(cfg))))


class Batch:
    """Device-resident lockstep batch: StochasticBatch (engine.hpp:250-266) whose members
    may each carry their own grid (n_grids == n_envs) or share one (n_grids == 1)."""

    def __init__(self, n_envs: int, height: int, width: int, device: int = 0, stream=None):
        self._h = C.c_void_p()
        check(lib().ebl_batch_create(C.byref(self._h), device, n_envs, height, width,
                                     C.c_void_p(stream) if stream else None))
        self.n_envs, self.height, self.width = n_envs, height, width

    # -- lifetime -----------------------------------------------------------------------
    def close(self):
        if self._h:
            lib().ebl_batch_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    # -- configuration --------------------------------------------------------------------
    def set_config(self, cfg) -> None:
        check(lib().ebl_batch_set_config(self._h, C.byref(as_config(cfg))))

    def set_grid(self, wind_speed, wind_direction, veg, den, slope8) -> None:
        """General GridState layers (grid.hpp:192-211): [G, H, W] (+ [.., 8] for slope)."""
        arrs = [np.ascontiguousarray(x, dtype=np.float64)
                for x in (wind_speed, wind_direction, veg, den, slope8)]
        n_grids = arrs[0].size // (self.height * self.width)
        check(lib().ebl_batch_set_grid(self._h, n_grids, *[_ptr(a) for a in arrs]))

    def set_terrain(self, fuel_class, elevation, class_veg, class_den, cellsize=30.0) -> None:
        """North-star layout: uint8 class [G,H,W] into a (veg, den) palette, fp32 elevation."""
        fc = np.ascontiguousarray(fuel_class, dtype=np.uint8)
        el = np.ascontiguousarray(elevation, dtype=np.float32)
        cv = np.ascontiguousarray(class_veg, dtype=np.float64)
        cd = np.ascontiguousarray(class_den, dtype=np.float64)
        n_grids = fc.size // (self.height * self.width)
        check(lib().ebl_batch_set_terrain(self._h, n_grids, _ptr(fc), _ptr(el), cv.size, _ptr(cv),
                                          _ptr(cd), float(cellsize)))

    def set_landcover(self, landcover, elevation, table, fallback=None, nodata_code=None,
                      cellsize=30.0) -> None:
        """grid_from_rasters / fuel_from_landcover (geodata.cpp:324-369) on the device.

        landcover: int codes [G,H,W]; elevation: fp32 [G,H,W] (NaN = DEM nodata);
        table: {code: (veg, den)}; fallback: (veg, den) for unknown codes or None."""
        lc = np.ascontiguousarray(landcover, dtype=np.int32)
        el = np.ascontiguousarray(elevation, dtype=np.float32)
        codes = np.ascontiguousarray(list(table.keys()), dtype=np.int32)
        veg = np.ascontiguousarray([v for v, _ in table.values()], dtype=np.float64)
        den = np.ascontiguousarray([d for _, d in table.values()], dtype=np.float64)
        n_grids = lc.size // (self.height * self.width)
        fb = (0.0, 0.0) if fallback is None else fallback
        check(lib().ebl_batch_set_landcover(
            self._h, n_grids, _ptr(lc), _ptr(el), int(nodata_code is not None),
            0 if nodata_code is None else int(nodata_code), codes.size, _ptr(codes), _ptr(veg),
            _ptr(den), int(fallback is not None), float(fb[0]), float(fb[1]), float(cellsize)))

    def synth_terrain(self, seed: int, env_id0: int = 0, elev_max: float = 500.0,
                      wind_max: float = 10.0, cellsize: float = 30.0) -> None:
        """The C1 generator run on the device (bit-identical to synth_terrain below)."""
        check(lib().ebl_batch_synth_terrain(self._h, seed, env_id0, float(elev_max), float(wind_max),
                                            float(cellsize)))

    def synth_ignitions(self, seed: int, count: int, env_id0: int = 0) -> int:
        """Seeded ignitions on the device into the state (bit-identical to synth_ignitions)."""
        placed = C.c_int()
        check(lib().ebl_batch_synth_ignitions(self._h, seed, env_id0, count, C.byref(placed)))
        return placed.value

    def get_terrain(self):
        """(fuel_class uint8 [G,H,W], elevation fp32 [G,H,W]) of the terrain form."""
        n = self.n_envs  # G = n_envs or 1; the C-ABI copies n_grids grids
        fc = np.zeros((n, self.height, self.width), np.uint8)
        el = np.zeros((n, self.height, self.width), np.float32)
        check(lib().ebl_batch_get_terrain(self._h, _ptr(fc), _ptr(el)))
        return fc, el

    def set_wind(self, speed, direction) -> None:
        sp = np.ascontiguousarray(np.atleast_1d(speed), dtype=np.float64)
        dr = np.ascontiguousarray(np.atleast_1d(direction), dtype=np.float64)
        check(lib().ebl_batch_set_wind(self._h, sp.size, _ptr(sp), _ptr(dr)))

    def set_kernel(self, which: int) -> None:
        check(lib().ebl_batch_set_kernel(self._h, which))

    def set_tiling(self, tile_h: int, tile_w: int = 0, halo: int = 0) -> None:
        """Explicit blocked-kernel tiling (tests); tile_h = 0 restores the planner."""
        check(lib().ebl_batch_set_tiling(self._h, tile_h, tile_w, halo))

    # -- state / key ----------------------------------------------------------------------
    def set_state(self, states) -> None:
        st = np.ascontiguousarray(np.broadcast_to(np.asarray(states, dtype=np.uint8),
                                                  (self.n_envs, self.height, self.width)))
        check(lib().ebl_batch_set_state(self._h, _ptr(st)))

    def get_state(self) -> np.ndarray:
        out = np.empty((self.n_envs, self.height, self.width), dtype=np.uint8)
        check(lib().ebl_batch_get_state(self._h, _ptr(out)))
        return out

    def state_device_ptr(self) -> int:
        return lib().ebl_batch_state_device_ptr(self._h)

    def set_key(self, seed: int, step: int = 0, streams=None, first_stream: int = 0) -> None:
        """StochasticBatch seed/step and member streams (make_stochastic_batch, engine.cpp:122-132)."""
        s = None if streams is None else np.ascontiguousarray(streams, dtype=np.uint64)
        check(lib().ebl_batch_set_key(self._h, seed, step, _ptr(s), first_stream))

    @property
    def step_index(self) -> int:
        return lib().ebl_batch_step_index(self._h)

    # -- stepping -------------------------------------------------------------------------
    def step(self, n_steps: int = 1) -> None:
        """step_batch (engine.cpp:134-159) n_steps times, asynchronously on the batch stream."""
        check(lib().ebl_step_batch(self._h, n_steps))

    def run(self, initial, n_steps: int, out=None) -> np.ndarray:
        """set_state(initial) + step(n_steps) + get_state() from/to host buffers, pipelined over
        env chunks (ebl_batch_run); pass pinned arrays for overlapped copies."""
        st = np.ascontiguousarray(np.broadcast_to(np.asarray(initial, dtype=np.uint8),
                                                  (self.n_envs, self.height, self.width)))
        shape = (self.n_envs, self.height, self.width)
        if out is None:
            out = np.empty(shape, dtype=np.uint8)
        elif (not isinstance(out, np.ndarray) or out.dtype != np.uint8 or out.shape != shape
              or not out.flags.c_contiguous or not out.flags.writeable):
            raise ValueError(f"out must be a writeable C-contiguous uint8 array of shape {shape}")
        check(lib().ebl_batch_run(self._h, _ptr(st), n_steps, _ptr(out)))
        return out

    def set_pipeline(self, chunks: int) -> None:
        check(lib().ebl_batch_set_pipeline(self._h, chunks))

    def snapshot_text(self, layers_dev: int | None = None, n_layers: int = 0, steps=None, agents=None) -> str:
        """serialize_snapshot (snapshot.cpp:55-70) of the batch's current layers (or n_layers device
        layers at layers_dev, e.g. a recorded trajectory), concatenated; steps [n] (default: the
        batch step); agents [n, 3] (row, col, water; row < 0: no agent line).  Rendered on the
        device."""
        n = self.n_envs if layers_dev is None else n_layers
        st = None if steps is None else np.ascontiguousarray(np.broadcast_to(steps, (n,)), dtype=np.uint64)
        ag = None if agents is None else np.ascontiguousarray(agents, dtype=np.int32).reshape(n, 3)
        ln = C.c_size_t()
        args = (self._h, layers_dev, n, _ptr(st), _ptr(ag))
        check(lib().ebl_batch_snapshot_text(*args, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(max(ln.value, 1))
        check(lib().ebl_batch_snapshot_text(*args, buf, ln.value, C.byref(ln)))
        return buf.raw[:ln.value].decode()

    def step_record(self, n_steps: int) -> np.ndarray:
        """step(n_steps) keeping every step's layers (run_stochastic record=true, engine.cpp:116):
        [n_steps, n_envs, H, W] uint8 (the initial layers are not included)."""
        out = np.empty((n_steps, self.n_envs, self.height, self.width), dtype=np.uint8)
        check(lib().ebl_step_batch_record(self._h, n_steps, _ptr(out), 0))
        return out

    def set_wind_schedule(self, speed, direction) -> None:
        """Terrain-form WindSchedule: speed/direction [n_sched, n_winds] (n_winds 1 or n_envs)."""
        sp = np.ascontiguousarray(np.atleast_2d(speed), dtype=np.float64)
        dr = np.ascontiguousarray(np.atleast_2d(direction), dtype=np.float64)
        check(lib().ebl_batch_set_wind_schedule(self._h, sp.shape[0], sp.shape[1], _ptr(sp), _ptr(dr)))

    def set_grid_wind_schedule(self, speed, direction) -> None:
        """General-form WindSchedule of per-cell WindFields: [n_sched, n_grids, H, W]."""
        sp = np.ascontiguousarray(speed, dtype=np.float64)
        dr = np.ascontiguousarray(direction, dtype=np.float64)
        check(lib().ebl_batch_set_grid_wind_schedule(self._h, sp.shape[0], _ptr(sp), _ptr(dr)))

    def sync(self) -> None:
        check(lib().ebl_batch_sync(self._h))

    def counts(self) -> np.ndarray:
        """[n_envs, 4] int32: unburned, burning, burned, newly ignited (fire_fraction_stats)."""
        out = np.empty((self.n_envs, 4), dtype=np.int32)
        check(lib().ebl_batch_counts(self._h, _ptr(out)))
        return out

    def fractions(self) -> np.ndarray:
        """fire_fraction_stats (engine.cpp:185-198) per env: [n_envs, 3] doubles."""
        c = self.counts()[:, :3].astype(np.float64)
        return c / float(self.height * self.width)

    def intensity(self, record_form: bool = True):
        """lambda and p_ignite (fp32) of the current layers; record_form: the slope-record form of
        the resident kernels, else the on-the-fly elevation form (terrain layers)."""
        lam = np.empty((self.n_envs, self.height, self.width), dtype=np.float32)
        p = np.empty_like(lam)
        check(lib().ebl_batch_intensity_form(self._h, int(record_form), _ptr(lam), _ptr(p)))
        return lam, p

    # -- deterministic mode (engine.hpp:147-245) + reverse-mode gradient (C4) ----------------
    def det_set_state(self, p_un, p_burn, p_bd) -> None:
        shp = (self.n_envs, self.height, self.width)
        arrs = [np.ascontiguousarray(np.broadcast_to(np.asarray(x, dtype=np.float64), shp))
                for x in (p_un, p_burn, p_bd)]
        check(lib().ebl_det_set_state(self._h, *[_ptr(a) for a in arrs]))

    def det_set_state_from_fire(self) -> None:
        check(lib().ebl_det_set_state_from_fire(self._h))

    def det_get_state(self):
        shp = (self.n_envs, self.height, self.width)
        out = [np.empty(shp, np.float64) for _ in range(3)]
        check(lib().ebl_det_get_state(self._h, *[_ptr(a) for a in out]))
        return tuple(out)

    def det_forward(self, n_steps: int, record: bool = True) -> None:
        check(lib().ebl_det_forward(self._h, n_steps, int(record)))

    def det_set_mask(self, mask) -> None:
        """Make the target burn mask resident (det_loss_grad(None, ...) then reuses it)."""
        m = np.ascontiguousarray(np.broadcast_to(np.asarray(mask, dtype=np.float64),
                                                 (self.n_envs, self.height, self.width)))
        check(lib().ebl_det_set_mask(self._h, _ptr(m)))

    def det_loss_grad(self, mask, bce_weight=0.0, mse_weight=1.0, pool=1):
        """(loss [n_envs], grad [n_envs, 6]) after a recorded det_forward (calibrate.hpp:120-146);
        mask None: the det_set_mask target."""
        m = None if mask is None else np.ascontiguousarray(
            np.broadcast_to(np.asarray(mask, dtype=np.float64), (self.n_envs, self.height, self.width)))
        loss = np.empty(self.n_envs, np.float64)
        grad = np.empty((self.n_envs, 6), np.float64)
        check(lib().ebl_det_loss_grad(self._h, _ptr(m), float(bce_weight), float(mse_weight), int(pool),
                                      _ptr(loss), _ptr(grad)))
        return loss, grad

    def calibrate(self, p_un, p_burn, p_bd, mask, horizon, iterations=300, init_theta=None,
                  optimize=None, lr=1e-2, max_horizon=2000, bce_weight=1.0, mse_weight=1.0, pool=4):
        """calibrate (calibrate.cpp:104-167) on the device; returns dict(loss_history,
        theta_history, best_theta, best_loss, initial_loss)."""
        o = _lib.CalibOptions()
        lib().ebl_default_calib_options(C.byref(o))
        o.iterations = iterations
        if init_theta is not None:
            o.init_theta = (C.c_double * 6)(*init_theta)
        if optimize is not None:
            o.optimize = (C.c_int * 6)(*[int(x) for x in optimize])
        o.lr, o.max_horizon = lr, max_horizon
        shp = (self.n_envs, self.height, self.width)
        planes = [np.ascontiguousarray(np.broadcast_to(np.asarray(x, dtype=np.float64), shp))
                  for x in (p_un, p_burn, p_bd, mask)]
        lh = np.empty(iterations + 1)
        th = np.empty((iterations + 1, 6))
        best = np.empty(6)
        bl = C.c_double()
        check(lib().ebl_calibrate(self._h, *[_ptr(a) for a in planes], horizon, float(bce_weight),
                                  float(mse_weight), int(pool), C.byref(o), _ptr(lh), _ptr(th),
                                  _ptr(best), C.byref(bl)))
        return dict(loss_history=lh, theta_history=th, best_theta=best, best_loss=bl.value,
                    initial_loss=lh[0])

    def diag(self, reset: bool = False) -> dict:
        out = np.zeros(4, dtype=np.uint64)
        t = np.zeros(2, dtype=np.uint64)
        check(lib().ebl_batch_tile_stats(self._h, _ptr(t), int(reset)))
        check(lib().ebl_batch_diag(self._h, _ptr(out), int(reset)))
        return {"fp64_fallbacks": int(out[0]), "ambiguous": int(out[1]), "steps": int(out[2]),
                "launches": int(out[3]), "tiles_processed": int(t[0]), "tiles_launched": int(t[1])}


# ---- one-shot reference signatures ----------------------------------------------------------
def _layers(grid):
    return [np.ascontiguousarray(grid[k], dtype=np.float64)
            for k in ("speed", "dir", "veg", "den", "slope8")]


def step_stochastic(fire, grid: dict, cfg, key) -> np.ndarray:
    """step_stochastic(fire, grid, cfg, RngKey{seed, step, stream}) (engine.hpp:204-207)."""
    fire = np.ascontiguousarray(fire, dtype=np.uint8)
    out = np.empty_like(fire)
    seed, step, stream = key
    check(lib().ebl_step_stochastic(fire.shape[0], fire.shape[1], _ptr(fire),
                                    *[_ptr(a) for a in _layers(grid)], C.byref(as_config(cfg)),
                                    seed, step, stream, _ptr(out)))
    return out


def run_stochastic(initial, grid: dict, cfg, key, steps: int) -> np.ndarray:
    """run_stochastic(initial, grid, cfg, key, steps).final_state (engine.hpp:215-217)."""
    fire = np.ascontiguousarray(initial, dtype=np.uint8)
    out = np.empty_like(fire)
    seed, step, stream = key
    check(lib().ebl_run_stochastic(fire.shape[0], fire.shape[1], _ptr(fire),
                                   *[_ptr(a) for a in _layers(grid)], C.byref(as_config(cfg)),
                                   seed, step, stream, steps, _ptr(out)))
    return out


# ---- inputs -----------------------------------------------------------------------------------
@dataclass
class Terrain:
    fuel_class: np.ndarray   # uint8 [n, H, W], palette index
    elevation: np.ndarray    # float32 [n, H, W], metres
    wind_speed: np.ndarray   # float64 [n]
    wind_direction: np.ndarray
    class_veg: np.ndarray    # float64 [11]
    class_den: np.ndarray
    cellsize: float = 30.0

    def veg(self) -> np.ndarray:
        return self.class_veg[self.fuel_class]

    def den(self) -> np.ndarray:
        return self.class_den[self.fuel_class]


def worldcover_palette():
    codes = np.empty(11, dtype=np.int32)
    veg = np.empty(11, dtype=np.float64)
    den = np.empty(11, dtype=np.float64)
    lib().ebl_worldcover_palette(_ptr(codes), _ptr(veg), _ptr(den))
    return codes, veg, den


def synth_terrain(seed: int, n_envs: int, height: int, width: int, env_id0: int = 0,
                  elev_max: float = 500.0, wind_max: float = 10.0) -> Terrain:
    """Seeded C1-style terrain."""
    fc = np.empty((n_envs, height, width), dtype=np.uint8)
    el = np.empty((n_envs, height, width), dtype=np.float32)
    ws = np.empty(n_envs, dtype=np.float64)
    wd = np.empty(n_envs, dtype=np.float64)
    check(lib().ebl_synth_terrain(seed, env_id0, n_envs, height, width, elev_max, wind_max,
                                  _ptr(fc), _ptr(el), _ptr(ws), _ptr(wd)))
    _, veg, den = worldcover_palette()
    return Terrain(fc, el, ws, wd, veg, den)


def synth_ignitions(seed: int, terrain: Terrain, count: int, env_id0: int = 0) -> np.ndarray:
    n, h, w = terrain.fuel_class.shape
    st = np.empty((n, h, w), dtype=np.uint8)
    check(lib().ebl_synth_ignitions(seed, env_id0, n, h, w, _ptr(terrain.fuel_class),
                                    _ptr(terrain.class_veg), _ptr(terrain.class_den), count,
                                    _ptr(st)))
    return st


# ---- RL -----------------------------------------------------------------------------------------
def default_preset() -> EnvConfig:
    c = EnvConfig()
    lib().ebl_env_default_preset(C.byref(c))
    return c


def smoke10_preset() -> EnvConfig:
    c = EnvConfig()
    lib().ebl_env_smoke10_preset(C.byref(c))
    return c


def observation_size(cfg: EnvConfig) -> int:
    return lib().ebl_env_observation_size(C.byref(cfg))


class VecFireEnv:
    """A batch of RL envs stepped on device.

    variant RL_REFERENCE: FireSuppressionEnv (rl_env.hpp:93-110) per env — reset/observe/step
    with the reference's Move x Valve actions, single-cell douse and reward.
    variant RL_TANKER: the BASELINE C2 air-tanker env ((x,y) actions, 3x3 extinguish + wet,
    reward = -newly ignited, auto-reset), terrain from `terrain`.
    """

    def __init__(self, n_envs: int, cfg: EnvConfig | None = None, variant: int = _lib.RL_REFERENCE,
                 terrain: Terrain | None = None, sim_cfg=None, ignitions: int = 5,
                 max_steps: int = 256, env_id0: int = 0, device: int = 0, stream=None):
        self.variant = variant
        if variant == _lib.RL_REFERENCE:
            self.cfg = cfg if cfg is not None else default_preset()
            h, w = self.cfg.height, self.cfg.width
        else:
            assert terrain is not None
            _, h, w = terrain.fuel_class.shape
            self.cfg = cfg
        self.batch = Batch(n_envs, h, w, device=device, stream=stream)
        if variant == _lib.RL_TANKER:
            self.batch.set_terrain(terrain.fuel_class, terrain.elevation, terrain.class_veg,
                                   terrain.class_den, terrain.cellsize)
            self.batch.set_wind(terrain.wind_speed, terrain.wind_direction)
            self.batch.set_config(sim_cfg)
        check(lib().ebl_rl_configure(self.batch.handle, variant,
                                     C.byref(self.cfg) if self.cfg is not None else None,
                                     ignitions, max_steps, env_id0))
        self.n_envs, self.height, self.width = n_envs, h, w

    def reset(self, seed: int, streams=None, mask=None) -> None:
        s = None if streams is None else np.ascontiguousarray(streams, dtype=np.uint64)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        check(lib().ebl_rl_reset(self.batch.handle, seed, _ptr(s), _ptr(m)))

    def step(self, actions=None):
        """Returns (reward [n] float64, done [n] uint8)."""
        a = None if actions is None else np.ascontiguousarray(actions, dtype=np.int32)
        reward = np.empty(self.n_envs, dtype=np.float64)
        done = np.empty(self.n_envs, dtype=np.uint8)
        check(lib().ebl_rl_step(self.batch.handle, _ptr(a), _ptr(reward), _ptr(done), 0))
        return reward, done

    def rollout(self, n_steps: int):
        rs = np.empty(self.n_envs, dtype=np.float64)
        ep = np.empty(self.n_envs, dtype=np.int32)
        check(lib().ebl_rl_rollout(self.batch.handle, n_steps, _ptr(rs), _ptr(ep)))
        return rs, ep

    def step_device(self, actions, reward, done) -> None:
        """One step with DEVICE tensors (a learner in the loop, no host round trip): actions int32
        [n] (row*W+col for the tanker; None: the device random policy), reward float64 [n] and
        done uint8 [n] written on the batch stream (ebl_rl_step device_io=1)."""
        for t, dt in ((actions, "int32"), (reward, "float64"), (done, "uint8")):
            if t is not None and (not t.is_cuda or str(t.dtype) != "torch." + dt or t.numel() != self.n_envs
                                  or not t.is_contiguous()):
                raise ValueError(f"expected a contiguous cuda {dt} tensor of {self.n_envs} elements")
        check(lib().ebl_rl_step(self.batch.handle, None if actions is None else C.c_void_p(actions.data_ptr()),
                                C.c_void_p(reward.data_ptr()), C.c_void_p(done.data_ptr()), 1))

    def observe_device(self, out) -> None:
        """Tanker observation into a device uint8 tensor [n, H, W]: FireState | wet << 2."""
        if not out.is_cuda or str(out.dtype) != "torch.uint8" or out.numel() != self.n_envs * self.height * self.width \
                or not out.is_contiguous():
            raise ValueError("expected a contiguous cuda uint8 tensor of n*H*W elements")
        check(lib().ebl_rl_observe_device(self.batch.handle, C.c_void_p(out.data_ptr())))

    def observe(self) -> np.ndarray:
        osz = observation_size(self.cfg)
        out = np.empty((self.n_envs, osz), dtype=np.float64)
        check(lib().ebl_rl_observe(self.batch.handle, _ptr(out)))
        return out

    def env_states(self):
        arr = (EnvState * self.n_envs)()
        check(lib().ebl_rl_get_env_states(self.batch.handle, arr))
        return list(arr)

    def set_env_states(self, states) -> None:
        arr = (EnvState * self.n_envs)(*states)
        check(lib().ebl_rl_set_env_states(self.batch.handle, arr))

    def fire(self) -> np.ndarray:
        return self.batch.get_state()

    def set_fire(self, states) -> None:
        self.batch.set_state(states)

    def wet(self) -> np.ndarray:
        out = np.empty((self.n_envs, self.height, self.width), dtype=np.uint8)
        check(lib().ebl_rl_get_wet(self.batch.handle, _ptr(out)))
        return out
