"""B200-native batched CA fire-spread step (drop-in for emberline's stochastic engine path).

The compute path is libember_b200.so (hand-written sm_100a kernels behind the C-ABI in
include/ember_b200.h); this package is its Python face.  See DESIGN.md.
"""
from ._lib import (CalibOptions, EmberError, EnvConfig, EnvState, InvalidArgument, LogicError,
                   FileError, NumericalError, OutOfRange,
                   RL_REFERENCE, RL_TANKER, SimConfig, lib)
from .engine import (BURNED, BURNING, KERNEL_AUTO, KERNEL_BLOCKED, KERNEL_WARP, KERNEL_RESIDENT, KERNEL_TILED, UNBURNED, Batch,
                     Terrain, VecFireEnv, as_config, default_config, default_preset,
                     host_buffer, observation_size, parse_snapshot, run_stochastic, smoke10_preset, step_stochastic,
                     synth_ignitions, synth_terrain, validate_config, worldcover_palette)

__all__ = [n for n in dir() if not n.startswith("_")]
