"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the CPU oracles.

* ``port()``  -> oracle/libember_oracle.so, the C restatement (ember_oracle.c), built from
  source anywhere (make -C oracle).
* ``ref()``   -> oracle/_ref/libebl_ref.so, the UNMODIFIED reference sources compiled in
  place (make -C oracle ref; only where /root/reference exists — the built .so travels).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module, and only as the checker or the CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libember_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libebl_ref.so")

_P, _I, _U64, _U32, _D = C.c_void_p, C.c_int, C.c_uint64, C.c_uint32, C.c_double


class EnvCfg(C.Structure):
    _fields_ = [("height", _I), ("width", _I), ("window_radius", _I), ("water_capacity", _I),
                ("burn_penalty", _D), ("max_episode_steps", _I), ("ignition_count", _I),
                ("waste_water", _I), ("wind_speed", _D), ("wind_direction", _D),
                ("fuel_veg", _D), ("fuel_den", _D), ("spread", _D * 6)]


class EnvSt(C.Structure):
    _fields_ = [("agent_row", _I), ("agent_col", _I), ("water", _I), ("step", _I),
                ("seed", _U64), ("stream", _U64), ("done", _I)]


class TankerCfg(C.Structure):
    _fields_ = [("ignitions", _I), ("max_steps", _I), ("autoreset", _I)]


class TankerSt(C.Structure):
    _fields_ = [("step", _I), ("episode", _U32), ("done", _I)]


def ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _bind(L, table):
    for name, (res, args) in table.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


_PORT_SIG = {
    "ebo_rng_word": (_U64, [_U64] * 5),
    "ebo_rng_uniform": (_D, [_U64] * 5),
    "ebo_rng_below": (_U64, [_U64] * 6),
    "ebo_wrap_angle": (_D, [_D]),
    "ebo_offset_angle": (_D, [_I]),
    "ebo_grid_layers": (_P, [_I, _I, _P, _P, _P, _P, _P]),
    "ebo_grid_terrain": (_P, [_I, _I, _P, _P, _P, _D, _D, _D]),
    "ebo_grid_free": (None, [_P]),
    "ebo_tables": (None, [_P, _P, _P, _P]),
    "ebo_intensity": (None, [_P, _P, _P, _P, _P]),
    "ebo_step_tables": (None, [_I, _I, _P, _P, _D, _U64, _U64, _U64, _P, _P]),
    "ebo_run": (None, [_P, _P, _U64, _U64, _U64, _I, _P]),
    "ebo_run_envs": (_D, [_P, _I, _P, _U64, _P, _I, _P, _I]),
    "ebo_counts": (None, [_P, _I, _P]),
    "ebo_env_obs_size": (_I, [C.POINTER(EnvCfg)]),
    "ebo_env_reset": (None, [C.POINTER(EnvCfg), _U64, _U64, C.POINTER(EnvSt), _P]),
    "ebo_env_step": (_I, [C.POINTER(EnvCfg), C.POINTER(EnvSt), _P, _I, C.POINTER(EnvSt), _P,
                          C.POINTER(_D), _P]),
    "ebo_env_observe": (None, [C.POINTER(EnvCfg), C.POINTER(EnvSt), _P, _P]),
    "ebo_random_policy": (_I, [_U64, _U64, _U64]),
    "ebo_tanker_reset": (None, [_P, C.POINTER(TankerCfg), _U64, _U32, _U32, C.POINTER(TankerSt),
                                _P, _P]),
    "ebo_tanker_step": (None, [_P, _P, _P, _D, C.POINTER(TankerCfg), _U64, _U32, _I,
                               C.POINTER(TankerSt), _P, _P, _P, _P]),
    "ebo_tanker_policy": (_I, [_U64, _U32, C.POINTER(TankerSt), _I]),
    "ebo_det_step_tables": (None, [_I, _I, _P, _P, _D, _P, _P, _P, _P, _P, _P]),
    "ebo_det_run": (None, [_P, _P, _I, _P, _P, _P]),
    "ebo_det_loss_grad": (None, [_P, _P, _I, _P, _P, _D, _D, _I, C.POINTER(_D), _P]),
    "ebo_calibrate": (_I, [_P, _P, _P, _P, _P, _I, _D, _D, _I, _I, _P, _P, _D, _P, _P, _P, C.POINTER(_D)]),
    "ebo_snapshot_text": (C.c_long, [_I, _I, _P, _U64, _I, _I, _I, C.c_char_p, C.c_long]),
    "ebo_synth_terrain": (None, [_U64, _U32, _I, _I, _I, _D, _D, _P, _P, _P, _P]),
    "ebo_worldcover_palette": (None, [_P, _P, _P]),
    "ebo_synth_ignitions": (_I, [_U64, _U32, _I, _I, _I, _P, _P, _P, _I, _P]),
    "ebo_tanker_run_envs": (_D, [_P, _I, _P, C.POINTER(TankerCfg), _U64, _U32, _P, _I, _I, C.POINTER(_D),
                                 _P, _P, _P, _P]),
}

_REF_SIG = {
    "ref_last_error": (C.c_char_p, []),
    "ref_rng_word": (_U64, [_U64] * 5),
    "ref_rng_uniform": (_D, [_U64] * 5),
    "ref_rng_below": (_U64, [_U64] * 6),
    "ref_grid_layers": (_P, [_I, _I, _P, _P, _P, _P, _P]),
    "ref_grid_terrain": (_P, [_I, _I, _P, _P, _P, _D, _D, _D]),
    "ref_grid_from_rasters": (_P, [_I, _I, _P, _P, _I, _P, _P, _P, _I, _D, _D, _D, _D, _D]),
    "ref_grid_fuel": (_I, [_P, _P, _P]),
    "ref_grid_free": (None, [_P]),
    "ref_grid_slope": (_I, [_P, _P]),
    "ref_tables": (_I, [_P, _P, _P, _P]),
    "ref_intensity": (_I, [_P, _P, _P, _P, _P]),
    "ref_run_stochastic": (_I, [_P, _P, _U64, _U64, _U64, _I, _I, _P, _P]),
    "ref_reference_step": (_I, [_P, _P, _U64, _U64, _U64, _P, _P]),
    "ref_step_batch": (_I, [_P, _P, _U64, _U64, _I, _I, _P, _P]),
    "ref_run_envs": (_D, [_P, _I, _P, _U64, _P, _I, _P, _I]),
    "ref_max_threads": (_I, []),
    "ref_loss_grad_envs": (_D, [_P, _I, _P, _I, _P, _P, _D, _D, _I, _P, _P, _I]),
    "ref_env_batch": (_D, [C.POINTER(EnvCfg), _I, _U64, _U64, _I, _I, C.POINTER(C.c_longlong), C.POINTER(_D)]),
    "ref_worldcover": (_I, [_I, C.POINTER(_D), C.POINTER(_D)]),
    "ref_env_preset": (_I, [_I, C.POINTER(EnvCfg)]),
    "ref_env_reset": (_I, [C.POINTER(EnvCfg), _U64, _U64, C.POINTER(EnvSt), _P]),
    "ref_env_step": (_I, [C.POINTER(EnvCfg), C.POINTER(EnvSt), _P, _I, C.POINTER(EnvSt), _P,
                          C.POINTER(_D), _P]),
    "ref_env_observe": (_I, [C.POINTER(EnvCfg), C.POINTER(EnvSt), _P, _P]),
    "ref_random_policy": (_I, [_U64, _U64, _U64]),
    "ref_run_deterministic": (_I, [_P, _P, _I, _P, _P, _P]),
    "ref_loss_grad": (_I, [_P, _P, _I, _P, _P, _D, _D, _I, C.POINTER(_D), _P]),
    "ref_calibrate": (_I, [_P, _P, _P, _P, _P, _I, _D, _D, _I, _I, _P, _P, _D, _P, _P, _P, C.POINTER(_D)]),
    "ref_serialize_snapshot": (C.c_long, [_I, _I, _P, _U64, _I, _I, _I, C.c_char_p, C.c_long]),
    "ref_parse_snapshot": (_I, [C.c_char_p, C.c_long, C.POINTER(_I), C.POINTER(_I), C.POINTER(_U64), _P, C.c_long,
                                _P, C.POINTER(_I)]),
}

_port = None
_ref = None


def build_port() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def port():
    """The C restatement; built on demand (gcc is in the image everywhere)."""
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO) or (os.path.getmtime(PORT_SO) <
                                           os.path.getmtime(os.path.join(HERE, "ember_oracle.c"))):
            build_port()
        _port = _bind(C.CDLL(PORT_SO), _PORT_SIG)
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference compiled in place; None when neither built nor buildable here."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            if not os.path.isdir("/root/reference/proj"):
                return None
            subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
        _ref = _bind(C.CDLL(REF_SO), _REF_SIG)
    return _ref


def cfg_array(cfg) -> np.ndarray:
    """(p_base, alpha_w1, alpha_w2, alpha_s, alpha_gamma, p_continue) as float64[6]."""
    if hasattr(cfg, "as_list"):
        cfg = cfg.as_list()
    return np.ascontiguousarray(np.asarray(cfg, dtype=np.float64)[:6])


DEFAULT_CFG = np.array([0.12, 0.2, 0.4, 1.0, 1.0, 0.6])


class Grid:
    """Owns an oracle grid handle (port or ref) built from layers or terrain."""

    def __init__(self, L, kind: str, handle):
        self.L, self.kind, self.h = L, kind, handle

    def __del__(self):
        try:
            (self.L.ebo_grid_free if self.kind == "port" else self.L.ref_grid_free)(self.h)
        except Exception:
            pass


def grid_layers(L, kind, speed, direction, veg, den, slope8) -> Grid:
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (speed, direction, veg, den, slope8)]
    h, w = arrs[0].shape
    fn = L.ebo_grid_layers if kind == "port" else L.ref_grid_layers
    g = fn(h, w, *[ptr(a) for a in arrs])
    assert g, "oracle rejected the grid"
    return Grid(L, kind, g)


def grid_terrain(L, kind, veg, den, elev, cellsize, speed, direction) -> Grid:
    v = np.ascontiguousarray(veg, dtype=np.float64)
    d = np.ascontiguousarray(den, dtype=np.float64)
    e = np.ascontiguousarray(elev, dtype=np.float32)
    h, w = v.shape
    fn = L.ebo_grid_terrain if kind == "port" else L.ref_grid_terrain
    g = fn(h, w, ptr(v), ptr(d), ptr(e), float(cellsize), float(speed), float(direction))
    assert g, "oracle rejected the grid"
    return Grid(L, kind, g)


def grid_from_rasters(L, elev, landcover, table: dict, fallback=None, cellsize=30.0, speed=0.0,
                      direction=0.0):
    """Reference grid_from_rasters (geodata.cpp:351-369) -> (Grid, veg, den), or raises
    RuntimeError carrying the reference's message (FileError / invalid_argument)."""
    e = np.ascontiguousarray(elev, dtype=np.float32)
    lc = np.ascontiguousarray(landcover, dtype=np.float64)
    h, w = e.shape
    codes = np.ascontiguousarray(list(table.keys()), dtype=np.int32)
    veg = np.ascontiguousarray([v for v, _ in table.values()], dtype=np.float64)
    den = np.ascontiguousarray([d for _, d in table.values()], dtype=np.float64)
    fb = (0.0, 0.0) if fallback is None else fallback
    g = L.ref_grid_from_rasters(h, w, ptr(e), ptr(lc), codes.size, ptr(codes), ptr(veg), ptr(den),
                                int(fallback is not None), float(fb[0]), float(fb[1]), float(cellsize),
                                float(speed), float(direction))
    if not g:
        raise RuntimeError(L.ref_last_error().decode())
    grid = Grid(L, "ref", g)
    v = np.empty((h, w))
    d = np.empty((h, w))
    L.ref_grid_fuel(g, ptr(v), ptr(d))
    return grid, v, d


def run(L, kind, grid: Grid, cfg, seed, step0, stream, steps, state) -> np.ndarray:
    st = np.ascontiguousarray(state, dtype=np.uint8).copy()
    c = cfg_array(cfg)
    if kind == "port":
        L.ebo_run(grid.h, ptr(c), seed, step0, stream, steps, ptr(st))
        return st
    out = np.empty_like(st)
    rc = L.ref_run_stochastic(grid.h, ptr(c), seed, step0, stream, steps, 0, ptr(st), ptr(out))
    assert rc == 0, L.ref_last_error()
    return out


def intensity(L, kind, grid: Grid, cfg, fire):
    f = np.ascontiguousarray(fire, dtype=np.uint8)
    lam = np.empty(f.shape, dtype=np.float64)
    p = np.empty(f.shape, dtype=np.float64)
    c = cfg_array(cfg)
    (L.ebo_intensity if kind == "port" else L.ref_intensity)(grid.h, ptr(c), ptr(f), ptr(lam), ptr(p))
    return lam, p


def tables(L, kind, grid: Grid, cfg, n):
    pot = np.empty(n * 8, dtype=np.float64)
    gam = np.empty(n, dtype=np.float64)
    c = cfg_array(cfg)
    (L.ebo_tables if kind == "port" else L.ref_tables)(grid.h, ptr(c), ptr(pot), ptr(gam))
    return pot, gam


def fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def calibrate(L, kind, grid: Grid, init_planes, mask, horizon, iterations, init_theta, optimize=None,
              lr=1e-2, bce_w=1.0, mse_w=1.0, pool=4):
    """calibrate (calibrate.cpp:104-167) on the port or the reference: (rc, loss_hist, theta_hist,
    best_theta, best_loss)."""
    un, bu, bd = [np.ascontiguousarray(x, dtype=np.float64) for x in init_planes]
    m = np.ascontiguousarray(mask, dtype=np.float64)
    th = np.ascontiguousarray(init_theta, dtype=np.float64)
    opt = np.ascontiguousarray(np.ones(6) if optimize is None else optimize, dtype=np.int32)
    lh = np.empty(iterations + 1)
    thh = np.empty((iterations + 1, 6))
    best = np.empty(6)
    bl = _D()
    fn = L.ebo_calibrate if kind == "port" else L.ref_calibrate
    rc = fn(grid.h, ptr(un), ptr(bu), ptr(bd), ptr(m), horizon, bce_w, mse_w, pool, iterations, ptr(th),
            ptr(opt), lr, ptr(lh), ptr(thh), ptr(best), bl)
    return rc, lh, thh, best, bl.value


def snapshot_text(L, kind, fire, step, agent=None) -> bytes:
    """serialize_snapshot of one layer through the port (kind "port") or the reference ("ref")."""
    fire = np.ascontiguousarray(fire, dtype=np.uint8)
    h, w = fire.shape
    ar, ac, wt = agent if agent is not None else (-1, 0, 0)
    fn = L.ebo_snapshot_text if kind == "port" else L.ref_serialize_snapshot
    n = fn(h, w, ptr(fire), step, ar, ac, wt, None, 0)
    buf = C.create_string_buffer(n)
    fn(h, w, ptr(fire), step, ar, ac, wt, buf, n)
    return buf.raw[:n]


class SynthTerrain:
    """The benchmark's synthetic inputs from the port (no product library): same fields as
    paper_2512_06102_b200.Terrain, bit-identical to ebl_synth_terrain (tests/test_oracle_pin.py)."""

    def __init__(self, seed, n_envs, h, w, env_id0=0, elev_max=500.0, wind_max=10.0):
        L = port()
        self.fuel_class = np.empty((n_envs, h, w), dtype=np.uint8)
        self.elevation = np.empty((n_envs, h, w), dtype=np.float32)
        self.wind_speed = np.empty(n_envs)
        self.wind_direction = np.empty(n_envs)
        L.ebo_synth_terrain(seed, env_id0, n_envs, h, w, elev_max, wind_max, ptr(self.fuel_class),
                            ptr(self.elevation), ptr(self.wind_speed), ptr(self.wind_direction))
        self.class_veg = np.empty(11)
        self.class_den = np.empty(11)
        L.ebo_worldcover_palette(None, ptr(self.class_veg), ptr(self.class_den))
        self.cellsize = 30.0
        self.seed, self.env_id0 = seed, env_id0

    def veg(self):
        return self.class_veg[self.fuel_class]

    def den(self):
        return self.class_den[self.fuel_class]

    def ignitions(self, count, seed=None):
        n, h, w = self.fuel_class.shape
        st = np.empty((n, h, w), dtype=np.uint8)
        port().ebo_synth_ignitions(self.seed if seed is None else seed, self.env_id0, n, h, w,
                                   ptr(self.fuel_class), ptr(self.class_veg), ptr(self.class_den),
                                   count, ptr(st))
        return st


def tanker_run_envs(terrain, env_ids, cfg, seed, steps, ignitions=5, max_steps=256, threads=0):
    """The C restatement of the C2 tanker env over the given env ids (OpenMP over envs): returns
    dict(fire, wet [n, h, w], reward [n], episodes [n], seconds)."""
    L = port()
    ids = np.ascontiguousarray(env_ids, dtype=np.uint32)
    n = ids.size
    _, h, w = terrain.fuel_class.shape
    grids = [grid_terrain(L, "port", terrain.class_veg[terrain.fuel_class[e]],
                          terrain.class_den[terrain.fuel_class[e]], terrain.elevation[e], terrain.cellsize,
                          terrain.wind_speed[e], terrain.wind_direction[e]) for e in ids]
    hs = (_P * n)(*[g.h for g in grids])
    fire = np.empty((n, h, w), np.uint8)
    wet = np.empty((n, h, w), np.uint8)
    rw = np.empty(n)
    ep = np.empty(n, np.int32)
    tc = TankerCfg(ignitions, max_steps, 1)
    secs = L.ebo_tanker_run_envs(hs, n, ptr(cfg_array(cfg)), C.byref(tc), seed, 0, ptr(ids), steps, threads,
                                 None, ptr(fire), ptr(wet), ptr(rw), ptr(ep))
    return dict(fire=fire, wet=wet, reward=rw, episodes=ep, seconds=secs)
