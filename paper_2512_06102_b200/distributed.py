"""Env-sharded multi-GPU helpers (one process per GPU, torch.distributed).

C1 / C2 need no exchange (envs are independent, streams = global env ids).  C4 (gradient-based
calibration) shards the envs of a batch over the ranks and then needs ONE reduction of the loss
and the 6-vector gradient (d loss / d {p_base, alpha_w1, alpha_w2, alpha_s, alpha_gamma,
p_continue}, calibrate.hpp:21-28).  The sum is taken in a fixed order (per env in rank order,
then over envs) so the result does not depend on the rank count: identical, bit for bit, to the
single-process sum over the same envs.
"""
from __future__ import annotations

import numpy as np


def env_range(rank: int, world: int, n_envs: int) -> tuple[int, int]:
    """[first, last) global env ids of a rank: contiguous, balanced, covering 0..n_envs-1."""
    per, extra = divmod(n_envs, world)
    first = rank * per + min(rank, extra)
    return first, first + per + (1 if rank < extra else 0)


def reduce_loss_grad(dist, loss_env, grad_env, n_envs: int):
    """Global (sum of losses, summed gradient [6]) from this rank's per-env loss [m] / grad [m, 6]
    (Batch.det_loss_grad of its env range).  all_gather of the per-env rows into global env order,
    then a sequential fp64 sum: rank-count independent and deterministic.  Works on gloo (CPU
    tensors) and NCCL (pass CUDA tensors' numpy copies; the payload is 7 doubles per env)."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    first, last = env_range(rank, world, n_envs)
    assert len(loss_env) == last - first
    rows = np.zeros((n_envs, 7), np.float64)
    rows[first:last, 0] = loss_env
    rows[first:last, 1:] = grad_env
    t = torch.from_numpy(rows)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    full = np.zeros((n_envs, 7), np.float64)
    for r in range(world):
        f, l = env_range(r, world, n_envs)
        full[f:l] = gathered[r].cpu().numpy()[f:l]
    return sum_loss_grad(full[:, 0], full[:, 1:])


def sum_loss_grad(loss_env, grad_env):
    """The fixed-order sum over envs (env 0 first) of per-env losses and gradients."""
    loss = 0.0
    grad = np.zeros(6, np.float64)
    for e in range(len(loss_env)):
        loss += float(loss_env[e])
        grad += grad_env[e]
    return loss, grad
