"""Shift sharding across GPUs (north_star: "the work shards by shift,
the principal recycle space U and AU are broadcast once per outer step").

Reading D3 makes all shifts of an outer step independent, so one exchange per outer
step suffices and the CG loop has no per-iteration communication:

  rank 0     builds U~ (seeds + Ritz at k = 0, [V_i1, X^(k-1)] after)
  broadcast  U~ (n_c x N doubles); A U~, E U~ column-split across the ranks, all-gathered
  all ranks  anchor QR + Grams, guesses and group blocks (deterministic, identical)
  each rank  batched deflated CG on ITS shifts (assignment below)
  allgather  X^(k), G^(k) (M x N each), iteration counts, L-curve norms
  all ranks  L-curve corner and IRN weights (identical)

Assignment: outer step 0 deals the ladder round-robin; later steps use the group-aware
LPT of group_lpt_assign on the previous step's per-shift iteration counts (the cost
model of SURVEY §8(e)), ties broken by shift index, so every rank computes the same
assignment.

Every device loop computes a shift independently of the batch it shares: the
cluster-per-shift loop trivially, the streaming lockstep loop (images beyond L2) by fixed
row ranges and double-double p.w partials, and U^T V by row chunks fixed by N
(DESIGN.md §4.2). So a G-rank run reproduces the 1-rank solutions and iteration counts
bit for bit (validated for C4 by tools/validate_multirank.sh; the tiled persistent loop
between those sizes is not covered by this guarantee).
This module holds only host logic and collectives; it works on CPU tensors under gloo
(tests) and on CUDA tensors under NCCL (bench).
"""
from __future__ import annotations

import numpy as np
import torch


def round_robin(M: int, world: int) -> list[list[int]]:
    return [list(range(r, M, world)) for r in range(world)]


def lpt_assign(costs, world: int) -> list[list[int]]:
    """Greedy longest-processing-time assignment: shifts in decreasing cost order go to
    the currently least-loaded rank (ties: lower rank). Each rank's list is sorted."""
    costs = np.asarray(costs, dtype=np.float64)
    order = sorted(range(len(costs)), key=lambda l: (-costs[l], l))
    load = [0.0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for l in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(l)
        load[r] += costs[l] + 1.0
    return [sorted(x) for x in out]


def group_lpt_assign(iters, groups, world: int, J: int = 12, S_ref: float = 80.0) -> list[list[int]]:
    """Group-aware assignment: a GPU holding shifts of a group re-reads that
    group's W, AW, EW (24|J| B/px) every lockstep iteration while any of them is active, so
    groups are kept apart. Cost model per shift-iteration: S_ref = 80 B/px of per-shift
    vectors; per GPU and group touched: the longest of its shifts x 24|J| B/px. GPUs go to
    the groups in proportion to the groups' predicted bytes (>= 1 each), shifts to the GPUs
    of their group by LPT; with fewer GPUs than groups, plain LPT. Deterministic."""
    iters = np.asarray(iters, dtype=np.float64)
    groups = np.asarray(groups)
    gids = sorted(set(groups.tolist()))
    if world < len(gids) or len(gids) < 2:
        return lpt_assign(iters, world)
    cost = {g: S_ref * float(np.sum(iters[groups == g] + 1)) + 24.0 * J * float(np.max(iters[groups == g]) + 1)
            for g in gids}
    total = sum(cost.values())
    # largest-remainder apportionment of the GPUs, at least one per group
    share = {g: max(1, int(np.floor(world * cost[g] / total))) for g in gids}
    while sum(share.values()) > world:
        g = max(gids, key=lambda x: (share[x], -cost[x]))
        share[g] -= 1
    rem = sorted(gids, key=lambda g: (-(world * cost[g] / total - share[g]), g))
    i = 0
    while sum(share.values()) < world:
        share[rem[i % len(rem)]] += 1
        i += 1
    out: list[list[int]] = []
    for g in gids:
        idx = [int(l) for l in np.nonzero(groups == g)[0]]
        sub = lpt_assign(iters[idx], share[g])
        out.extend([[idx[j] for j in o] for o in sub])
    return [sorted(o) for o in out]


def assignment(k: int, M: int, world: int, prev_iters=None, groups=None, J: int = 12) -> list[list[int]]:
    if world == 1:
        return [list(range(M))]
    if k == 0 or prev_iters is None:
        return round_robin(M, world)
    if groups is not None:
        return group_lpt_assign(prev_iters, groups, world, J)
    return lpt_assign(prev_iters, world)


class Dist:
    """Thin wrapper over torch.distributed (None => single rank)."""

    def __init__(self, enabled: bool = False):
        self.enabled = enabled
        if enabled:
            import torch.distributed as dist
            self.d = dist
            self.rank = dist.get_rank()
            self.world = dist.get_world_size()
            # gloo (CPU tests, several ranks on one device) stages CUDA tensors through host
            self.host_comm = dist.get_backend() == "gloo"
        else:
            self.d = None
            self.rank, self.world = 0, 1
            self.host_comm = False

    def _dev(self, t):
        return t.cpu() if (self.host_comm and t.is_cuda) else t

    def barrier(self):
        if self.enabled:
            self.d.barrier()

    def bcast(self, t: torch.Tensor, src: int = 0) -> torch.Tensor:
        if self.enabled:
            c = self._dev(t)
            self.d.broadcast(c, src=src)
            if c is not t:
                t.copy_(c)
        return t

    def bcast_int(self, v: int, device) -> int:
        if not self.enabled:
            return int(v)
        t = torch.tensor([int(v)], dtype=torch.int64, device="cpu" if self.host_comm else device)
        self.d.broadcast(t, src=0)
        return int(t.item())

    def gather_rows(self, local: torch.Tensor, owners: list[list[int]], M: int) -> torch.Tensor:
        """All-gather row blocks: rank r holds rows owners[r] (in order) of an M-row
        matrix; returns the full matrix in global row order on every rank."""
        if not self.enabled:
            full = torch.empty((M,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
            full[owners[0]] = local
            return full
        mx = max(len(o) for o in owners)
        cdev = torch.device("cpu") if (self.host_comm and local.is_cuda) else local.device
        pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=cdev)
        if local.shape[0]:
            pad[:local.shape[0]] = local.to(cdev)
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        self.d.all_gather(bufs, pad)
        bufs = [b.to(local.device) for b in bufs]
        full = torch.empty((M,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        for r, o in enumerate(owners):
            if o:
                full[o] = bufs[r][:len(o)]
        return full

    def gather_np(self, local: np.ndarray, owners: list[list[int]], M: int, device) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64)).reshape(len(local), -1)
        full = self.gather_rows(t.to(device), owners, M)
        return full.cpu().numpy().reshape((M,) + local.shape[1:])
