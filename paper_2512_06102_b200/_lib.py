"""ctypes binding of the C-ABI in include/ember_b200.h (libember_b200.so).

This is the Python face of the same boundary the C++ drop-in
(include/emberline_b200.hpp) wraps.  There is deliberately no fallback: if the
CUDA library is missing, importing the product fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# EBL_LIB overrides the library path (A/B timing of two builds of the same ABI)
LIB_PATH = os.environ.get("EBL_LIB") or os.path.join(_HERE, "libember_b200.so")

EBL_OK, EBL_EINVAL, EBL_ELOGIC, EBL_ERANGE, EBL_ECUDA, EBL_ESTATE, EBL_ENUMERIC, EBL_EFILE = \
    0, -1, -2, -3, -4, -5, -6, -7
RL_REFERENCE, RL_TANKER = 0, 1


class SimConfig(C.Structure):
    """BasicSimConfig<double> (reference grid.hpp:171-180)."""

    _fields_ = [("p_base", C.c_double), ("alpha_w1", C.c_double), ("alpha_w2", C.c_double),
                ("alpha_s", C.c_double), ("alpha_gamma", C.c_double), ("p_continue", C.c_double),
                ("max_steps", C.c_int)]

    def as_list(self):
        return [self.p_base, self.alpha_w1, self.alpha_w2, self.alpha_s, self.alpha_gamma,
                self.p_continue]


class EnvConfig(C.Structure):
    """EnvConfig (reference rl_env.hpp:24-40)."""

    _fields_ = [("height", C.c_int), ("width", C.c_int), ("window_radius", C.c_int),
                ("water_capacity", C.c_int), ("burn_penalty", C.c_double),
                ("max_episode_steps", C.c_int), ("ignition_count", C.c_int),
                ("waste_water", C.c_int), ("wind_speed", C.c_double),
                ("wind_direction", C.c_double), ("fuel_veg", C.c_double),
                ("fuel_den", C.c_double), ("spread", SimConfig)]


class EnvState(C.Structure):
    """EnvState minus the fire layer (reference rl_env.hpp:67-75)."""

    _fields_ = [("agent_row", C.c_int32), ("agent_col", C.c_int32), ("water", C.c_int32),
                ("step", C.c_int32), ("seed", C.c_uint64), ("stream", C.c_uint64),
                ("done", C.c_int32), ("episode", C.c_uint32)]


class CalibOptions(C.Structure):
    """CalibrationOptions (reference calibrate.hpp:158-166)."""

    _fields_ = [("iterations", C.c_int), ("init_theta", C.c_double * 6), ("optimize", C.c_int * 6),
                ("lr", C.c_double), ("max_horizon", C.c_int)]


class EmberError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(EmberError, ValueError):   # std::invalid_argument
    pass


class LogicError(EmberError):                    # std::logic_error
    pass


class OutOfRange(EmberError, IndexError):        # std::out_of_range
    pass


class NumericalError(EmberError, ArithmeticError):  # emberline::NumericalError
    pass


class FileError(EmberError):                      # emberline::FileError
    pass


_EXC = {EBL_EINVAL: InvalidArgument, EBL_ELOGIC: LogicError, EBL_ERANGE: OutOfRange,
        EBL_ENUMERIC: NumericalError, EBL_EFILE: FileError}

_P = C.c_void_p
_I, _U64, _U32, _D = C.c_int, C.c_uint64, C.c_uint32, C.c_double

# name -> (restype, argtypes); every symbol include/ember_b200.h declares.
SIGNATURES = {
    "ebl_abi_version": (_I, []),
    "ebl_last_error": (C.c_char_p, []),
    "ebl_validate_config": (_I, [C.POINTER(SimConfig)]),
    "ebl_default_config": (None, [C.POINTER(SimConfig)]),
    "ebl_batch_create": (_I, [C.POINTER(_P), _I, _I, _I, _I, _P]),
    "ebl_batch_destroy": (None, [_P]),
    "ebl_batch_set_config": (_I, [_P, C.POINTER(SimConfig)]),
    "ebl_batch_set_grid": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "ebl_batch_set_terrain": (_I, [_P, _I, _P, _P, _I, _P, _P, _D]),
    "ebl_batch_set_landcover": (_I, [_P, _I, _P, _P, _I, C.c_int32, _I, _P, _P, _P, _I, _D, _D, _D]),
    "ebl_batch_synth_terrain": (_I, [_P, _U64, _U32, _D, _D, _D]),
    "ebl_batch_synth_ignitions": (_I, [_P, _U64, _U32, _I, C.POINTER(_I)]),
    "ebl_batch_get_terrain": (_I, [_P, _P, _P]),
    "ebl_batch_set_wind": (_I, [_P, _I, _P, _P]),
    "ebl_batch_set_state": (_I, [_P, _P]),
    "ebl_batch_get_state": (_I, [_P, _P]),
    "ebl_batch_set_state_device": (_I, [_P, _P]),
    "ebl_batch_get_state_device": (_I, [_P, _P]),
    "ebl_batch_state_device_ptr": (_P, [_P]),
    "ebl_batch_set_key": (_I, [_P, _U64, _U64, _P, _U64]),
    "ebl_batch_step_index": (_U64, [_P]),
    "ebl_step_batch": (_I, [_P, _I]),
    "ebl_batch_run": (_I, [_P, _P, _I, _P]),
    "ebl_batch_intensity_form": (_I, [_P, _I, _P, _P]),
    "ebl_batch_set_band": (_I, [_P, _I, _I]),
    "ebl_shards_step": (_I, [_P, _I, _I, _I]),
    "ebl_batch_set_profiling": (_I, [_P, _I]),
    "ebl_batch_profile": (_I, [_P, _P]),
    "ebl_batch_set_pipeline": (_I, [_P, _I]),
    "ebl_batch_set_kernel": (_I, [_P, _I]),
    "ebl_step_batch_record": (_I, [_P, _I, _P, _I]),
    "ebl_batch_set_wind_schedule": (_I, [_P, _I, _I, _P, _P]),
    "ebl_batch_set_grid_wind_schedule": (_I, [_P, _I, _P, _P]),
    "ebl_batch_set_tiling": (_I, [_P, _I, _I, _I]),
    "ebl_batch_set_row_offset": (_I, [_P, C.c_int64]),
    "ebl_batch_copy_rows": (_I, [_P, _I, _P, _I, _I]),
    "ebl_batch_rows_device": (_I, [_P, _I, _I, _P, _I]),
    "ebl_batch_counts": (_I, [_P, _P]),
    "ebl_batch_intensity": (_I, [_P, _P, _P]),
    "ebl_batch_diag": (_I, [_P, _P, _I]),
    "ebl_batch_tile_stats": (_I, [_P, _P, _I]),
    "ebl_rl_observe_device": (_I, [_P, _P]),
    "ebl_batch_set_det_tables": (_I, [_P, _I]),
    "ebl_batch_sync": (_I, [_P]),
    "ebl_device_rng_words": (_I, [_I, _P, _P]),
    "ebl_step_stochastic": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, C.POINTER(SimConfig), _U64,
                                 _U64, _U64, _P]),
    "ebl_run_stochastic": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, C.POINTER(SimConfig), _U64,
                                _U64, _U64, _I, _P]),
    "ebl_det_set_state": (_I, [_P, _P, _P, _P]),
    "ebl_det_set_state_from_fire": (_I, [_P]),
    "ebl_det_get_state": (_I, [_P, _P, _P, _P]),
    "ebl_det_forward": (_I, [_P, _I, _I]),
    "ebl_det_set_mask": (_I, [_P, _P]),
    "ebl_det_loss_grad": (_I, [_P, _P, _D, _D, _I, _P, _P]),
    "ebl_default_calib_options": (None, [C.POINTER(CalibOptions)]),
    "ebl_calibrate": (_I, [_P, _P, _P, _P, _P, _I, _D, _D, _I, C.POINTER(CalibOptions), _P, _P, _P,
                           C.POINTER(_D)]),
    "ebl_env_default_preset": (None, [C.POINTER(EnvConfig)]),
    "ebl_env_smoke10_preset": (None, [C.POINTER(EnvConfig)]),
    "ebl_env_observation_size": (_I, [C.POINTER(EnvConfig)]),
    "ebl_rl_configure": (_I, [_P, _I, C.POINTER(EnvConfig), _I, _I, _U32]),
    "ebl_rl_reset": (_I, [_P, _U64, _P, _P]),
    "ebl_rl_step": (_I, [_P, _P, _P, _P, _I]),
    "ebl_rl_rollout": (_I, [_P, _I, _P, _P]),
    "ebl_rl_observe": (_I, [_P, _P]),
    "ebl_rl_get_env_states": (_I, [_P, _P]),
    "ebl_rl_set_env_states": (_I, [_P, _P]),
    "ebl_rl_get_wet": (_I, [_P, _P]),
    "ebl_batch_snapshot_text": (_I, [_P, _P, _I, _P, _P, _P, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ebl_snapshot_parse": (_I, [C.c_char_p, C.c_size_t, C.POINTER(_I), C.POINTER(_I), C.POINTER(_U64), _P,
                                C.c_size_t, _P, C.POINTER(_I)]),
    "ebl_host_alloc": (_I, [C.c_size_t, C.POINTER(_P)]),
    "ebl_host_free": (_I, [_P]),
    "ebl_synth_terrain": (_I, [_U64, _U32, _I, _I, _I, _D, _D, _P, _P, _P, _P]),
    "ebl_worldcover_palette": (None, [_P, _P, _P]),
    "ebl_synth_ignitions": (_I, [_U64, _U32, _I, _I, _I, _P, _P, _P, _I, _P]),
}

_lib = None


def lib():
    """Load libember_b200.so once; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("EBL_LIB") and not hasattr(L, name):
                continue  # A/B runs against an older build (scripts/ab_*.sh): bind what it has
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != EBL_OK:
        msg = lib().ebl_last_error().decode(errors="replace")
        raise _EXC.get(rc, EmberError)(rc, msg)
