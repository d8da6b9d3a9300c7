"""Row-sharded single landscape (BASELINE C3): one H x W grid split into G row bands.

Each shard keeps its band plus K light-cone halo rows on each side that are not a global
edge, as an independent device batch whose RNG row offset is the global row of its first
layer row, so every cell draws with its global index (row*W + col, engine.cpp:17) and the
sharded trajectory is bit-identical to the unsharded one.  A run advances every shard K
steps (one launch of the blocked kernel: the halo is exactly the light cone), then swaps
K boundary rows with each neighbour:

  * single process, G devices (or G shards on one device for testing): `ShardedLandscape`;
    fused=True (default): ebl_shards_step, the exchange fused into the kernels -- each launch
    stores the rows its neighbours hold as halo straight into their layers (peer stores over
    NVLink), neighbours ordered by stream events, no host synchronisation; fused=False: a launch
    per shard then ebl_batch_copy_rows (cudaMemcpyPeerAsync) per halo;
  * one process per GPU: `exchange_halos` on torch.distributed (NCCL send/recv of the K-row
    halo tensors; gloo on CPU in tests).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib
from .engine import Batch, Terrain


@dataclass(frozen=True)
class Shard:
    band: tuple   # global rows [b0, b1) owned (written back) by this shard
    rows: tuple   # global rows [g0, g1) held in its layer (band + halos)

    @property
    def halo_top(self) -> int:      # rows of halo below the band (south side, lower rows)
        return self.band[0] - self.rows[0]

    @property
    def halo_bottom(self) -> int:   # rows of halo above the band (north side, higher rows)
        return self.rows[1] - self.band[1]


def plan_shards(height: int, n_shards: int, halo: int) -> list[Shard]:
    """Balanced row bands; halos of `halo` rows where a neighbour exists."""
    if n_shards < 1 or n_shards > height:
        raise ValueError("need 1 <= n_shards <= height")
    cuts = [round(i * height / n_shards) for i in range(n_shards + 1)]
    out = []
    for s in range(n_shards):
        b0, b1 = cuts[s], cuts[s + 1]
        out.append(Shard((b0, b1), (max(0, b0 - halo), min(height, b1 + halo))))
    return out


def halo_copies(shards: list[Shard]) -> list[tuple]:
    """(dst_shard, dst_row, src_shard, src_row, n_rows) in layer-local rows: every halo row of
    every shard is refreshed from the shard that owns it."""
    out = []
    for d, sh in enumerate(shards):
        for n_rows, g_first in ((sh.halo_top, sh.rows[0]), (sh.halo_bottom, sh.band[1])):
            if n_rows == 0:
                continue
            owner = d - 1 if g_first < sh.band[0] else d + 1
            src = shards[owner]
            out.append((d, g_first - sh.rows[0], owner, g_first - src.rows[0], n_rows))
    return out


class ShardedLandscape:
    """C3 driver: G shards on `devices` (default: all on device 0) of one terrain."""

    def __init__(self, terrain: Terrain, n_shards: int, devices=None, halo: int = 16, cfg=None,
                 fused: bool = True):
        assert terrain.fuel_class.shape[0] == 1, "one landscape"
        _, self.height, self.width = terrain.fuel_class.shape
        self.halo = halo
        self.fused = fused
        self.shards = plan_shards(self.height, n_shards, halo)
        self.copies = halo_copies(self.shards)
        devices = devices or [0] * n_shards
        self.batches = []
        for sh, dev in zip(self.shards, devices):
            g0, g1 = sh.rows
            b = Batch(1, g1 - g0, self.width, device=dev)
            b.set_terrain(terrain.fuel_class[:, g0:g1], terrain.elevation[:, g0:g1],
                          terrain.class_veg, terrain.class_den, terrain.cellsize)
            b.set_wind(terrain.wind_speed[:1], terrain.wind_direction[:1])
            b.set_config(cfg)
            check(lib().ebl_batch_set_row_offset(b.handle, g0))
            if g1 - g0 < self.height:  # halo tiles: never more steps per launch than halo rows
                b.set_tiling(min(32, g1 - g0), min(128, -(-self.width // 32) * 32), halo)
            check(lib().ebl_batch_set_band(b.handle, sh.band[0] - g0, sh.band[1] - g0))
            self.batches.append(b)
        self._handles = (C.c_void_p * len(self.batches))(*[b.handle.value for b in self.batches])

    def set_state(self, state: np.ndarray) -> None:
        state = np.asarray(state, dtype=np.uint8).reshape(self.height, self.width)
        for sh, b in zip(self.shards, self.batches):
            b.set_state(state[sh.rows[0]:sh.rows[1]])

    def get_state(self) -> np.ndarray:
        out = np.empty((self.height, self.width), np.uint8)
        for sh, b in zip(self.shards, self.batches):
            layer = b.get_state()[0]
            out[sh.band[0]:sh.band[1]] = layer[sh.halo_top:sh.halo_top + sh.band[1] - sh.band[0]]
        return out

    def set_key(self, seed: int, step: int = 0, stream: int = 0) -> None:
        for b in self.batches:
            b.set_key(seed, step, streams=[stream])

    def exchange(self) -> None:
        for d, drow, s, srow, n in self.copies:
            check(lib().ebl_batch_copy_rows(self.batches[d].handle, drow, self.batches[s].handle, srow, n))

    def step(self, n_steps: int) -> None:
        if self.fused:
            check(lib().ebl_shards_step(self._handles, len(self.batches), n_steps, self.halo))
            return
        done = 0
        while done < n_steps:
            k = min(self.halo, n_steps - done) if len(self.batches) > 1 else n_steps - done
            for b in self.batches:   # launches are async: shards on different GPUs overlap
                b.step(k)
            if len(self.batches) > 1:
                self.exchange()
            done += k

    def sync(self) -> None:
        for b in self.batches:
            b.sync()


def exchange_halos(dist, rank: int, shards: list[Shard], get_rows, set_rows, make_buffer) -> None:
    """One halo swap between ranks (one shard per rank) over torch.distributed.
    get_rows(row0, n) -> tensor of rows owned here; set_rows(row0, tensor) writes halo rows;
    make_buffer(n) -> receive tensor.  Rows are layer-local.  Deadlock-free ordering:
    all sends/recvs are posted non-blocking and then waited."""
    me = shards[rank]
    reqs, recvs = [], []
    for nb in (rank - 1, rank + 1):
        if nb < 0 or nb >= len(shards):
            continue
        other = shards[nb]
        # rows of my band the neighbour holds as halo
        lo, hi = max(me.band[0], other.rows[0]), min(me.band[1], other.rows[1])
        if hi > lo:
            reqs.append(dist.isend(get_rows(lo - me.rows[0], hi - lo), dst=nb))
        # rows of the neighbour's band I hold as halo
        lo, hi = max(other.band[0], me.rows[0]), min(other.band[1], me.rows[1])
        if hi > lo:
            buf = make_buffer(hi - lo)
            reqs.append(dist.irecv(buf, src=nb))
            recvs.append((lo - me.rows[0], buf))
    for r in reqs:
        r.wait()
    for row0, buf in recvs:
        set_rows(row0, buf)
