"""Tournament touch points of the pod hot path (SURVEY.md §8e, configs[3]).

One pod population per GPU; once per generation every rank contributes its
pods' (score, seq, pod_id), the board is ranked identically on every rank by
(score desc, seq asc) -- the order sequential ``leaderboard_update`` insertion
produces (tournament.hpp:104-119, test_tournament.cpp:95-126) -- and the top-k
elites' weights are broadcast from their owner ranks (the elite copy of
``generate_pod_init``, tournament.hpp:146-159).

Device path: ``prb_leaderboard_allgather_rank`` (NCCL all-gather + ranking
kernel) and ``prb_agent_broadcast`` (NCCL broadcast of params/m/v/t).  The
host helpers below only do bookkeeping (sequence numbers, which rank owns an
elite); they are what the CPU (gloo) tests exercise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

from . import _lib


def arrival_seq(generation: int, global_pod_id: int, total_pods: int) -> int:
    """Deterministic arrival order across ranks: the reference assigns seq on
    insertion (tournament.hpp:108); pods of one generation arrive in pod-id order."""
    return generation * total_pods + global_pod_id


def global_pod_id(rank: int, local: int, pods_per_rank: int) -> int:
    return rank * pods_per_rank + local


def owner_rank(pod_id: int, pods_per_rank: int) -> int:
    return pod_id // pods_per_rank


def rank_candidates_host(scores: Sequence[float], seqs: Sequence[int], capacity: int) -> List[int]:
    """Reference ordering as a specification (sort by score desc, seq asc, keep
    `capacity`); used by the CPU tests to check the bookkeeping, never on the
    device path."""
    idx = sorted(range(len(scores)), key=lambda i: (-scores[i], seqs[i]))
    return idx[:capacity]


@dataclass
class BoardEntry:
    score: float
    seq: int
    pod_id: int


class Communicator:
    """NCCL communicator owned by libprb (one per rank).  The 128-byte NCCL id
    is created on rank 0 and shared through ``share_id`` (e.g. a
    torch.distributed broadcast)."""

    def __init__(self, ctx, rank: int, world: int, share_id):
        self.ctx, self.rank, self.world = ctx, rank, world
        lib = _lib.lib()
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            lib.prb_comm_unique_id(uid)
        uid_bytes = share_id(bytes(uid))
        uid = (C.c_uint8 * 128)(*uid_bytes)
        h = C.c_void_p()
        lib.prb_comm_init(ctx.h, uid, world, rank, C.byref(h))
        self.h = h
        self.lib = lib

    def close(self):
        if self.h:
            self.lib.prb_comm_destroy(self.h)
            self.h = None


def allgather_rank(comm: Communicator, scores: Sequence[float], seqs: Sequence[int], ids: Sequence[int],
                   capacity: int) -> Tuple[List[BoardEntry], np.ndarray]:
    """Device all-gather of every rank's candidates + identical ranking on every rank."""
    from .podracer import DeviceArray
    ctx = comm.ctx
    n = len(scores)
    world = comm.world
    d_s = DeviceArray.from_numpy(ctx, np.asarray(scores, dtype=np.float64))
    d_q = DeviceArray.from_numpy(ctx, np.asarray(seqs, dtype=np.uint64))
    d_i = DeviceArray.from_numpy(ctx, np.asarray(ids, dtype=np.int64))
    a_s = DeviceArray(ctx, (world * n,), np.float64)
    a_q = DeviceArray(ctx, (world * n,), np.uint64)
    a_i = DeviceArray(ctx, (world * n,), np.int64)
    order = DeviceArray(ctx, (capacity + 1,), np.int32)
    comm.lib.prb_leaderboard_allgather_rank(comm.h, d_s.ptr, d_q.ptr, d_i.ptr, n, capacity, a_s.ptr, a_q.ptr, a_i.ptr,
                                            order.ptr, order.ptr + 4 * capacity)
    o = order.numpy()
    count = int(o[capacity])
    s, q, i = a_s.numpy(), a_q.numpy(), a_i.numpy()
    board = [BoardEntry(float(s[k]), int(q[k]), int(i[k])) for k in o[:count]]
    return board, o[:count]


def broadcast_agent(comm: Communicator, agent, root: int):
    """Elite weights (params, Adam m/v, t) from their owner rank to every rank."""
    comm.lib.prb_agent_broadcast(comm.h, agent.h, root)
