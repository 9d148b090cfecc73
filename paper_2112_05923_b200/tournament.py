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


class PodPopulation:
    """One GPU's pod population (BASELINE configs[3]): the tournament of tournament.hpp:395-506 run
    as synchronous generations, every pod's data on the device.

    Per generation (``generation``):
      1. worker_collect of every pod in ONE tcgen05 launch (prb_rollout_collect_pods: per-pod
         weights, a grouped GEMM; pod.hpp:408-433);
      2. every pod's ``learners`` PPO learners in ONE tensor-core launch, 8 co-resident CTAs
         per learner (prb_ppo_update_learners; pod.hpp:436-461), then fuse_parameters per pod
         (pod.hpp:141-172) into the pod's agent;
      3. evaluate every pod in one pass (prb_evaluate_pods: ``eval_episodes`` episodes per pod as
         one VecEnv, policy mean; pod.hpp:43-83) -> its score;
      4. the leaderboard: every rank's (score, seq, pod_id) all-gathered over NCCL and ranked
         identically on every rank (prb_leaderboard_allgather_rank; tournament.hpp:104-119), or
         ranked on the device alone with one rank;
      5. the next generation's pod inits (generate_pod_init tournament.hpp:136-162): a pod is
         fresh with probability ``fresh_prob`` (artifact_init), else a copy of one of the top_k
         elites -- broadcast from its owner rank (prb_agent_broadcast) -- mutated on the device
         (prb_agent_mutate, t := 0).  Decisions draw from a per-rank numpy generator; the weights
         never leave HBM.
    Scores, seqs and ids are the only host traffic.
    """

    def __init__(self, ctx, market, stock_cfg, pods: int, envs_per_pod: int, horizon: int, learners: int,
                 ppo_cfg, window=(0, None), eval_episodes: int = 10, eval_window=None, capacity: int = 10,
                 top_k: int = 3, fresh_prob: float = 0.2, sigma: float = 0.01, seed: int = 2112, rank: int = 0,
                 world: int = 1, comm: "Communicator" = None, state_dim: int = 181, action_dim: int = 30):
        from . import podracer as pr
        self.pr, self.ctx, self.rank, self.world, self.comm = pr, ctx, rank, world, comm
        self.P, self.L, self.cfg = pods, learners, ppo_cfg
        self.capacity, self.top_k, self.fresh_prob, self.sigma = capacity, top_k, fresh_prob, sigma
        self.S, self.A, self.seed = state_dim, action_dim, seed
        T = market.T if hasattr(market, "T") else None
        start, end = window
        if end is None:
            end = (T - 1) if T else 2047
        ew = eval_window or (start, end)
        self.envs = [pr.VectorizedEnvironment.stock(ctx, market, stock_cfg, start, end, envs_per_pod)
                     for _ in range(pods)]
        self.eval_envs = [pr.VectorizedEnvironment.stock(ctx, market, stock_cfg, ew[0], ew[1], eval_episodes)
                          for _ in range(pods)]
        for p, e in enumerate(self.envs):
            e.reset(pr.derive_seed(seed, 1, self.global_id(p)))
        self.rollouts = [pr.Rollout.for_env(e, horizon) for e in self.envs]
        self.agents = [pr.Agent.init(ctx, state_dim, action_dim, seed=pr.derive_seed(seed, 5, self.global_id(p)))
                       for p in range(pods)]
        self.learner_out = [[pr.Agent(ctx, state_dim, action_dim) for _ in range(learners)] for _ in range(pods)]
        self.elites = [pr.Agent(ctx, state_dim, action_dim) for _ in range(top_k)]
        self.rng = np.random.default_rng(seed * 7919 + rank)
        self.board: List[BoardEntry] = []
        self.gen = 0
        self.last_scores = None

    def global_id(self, p: int) -> int:
        return global_pod_id(self.rank, p, self.P)

    def generation(self) -> dict:
        pr = self.pr
        g = self.gen
        # 1. every pod's collect in one launch
        pr.collect_pods(self.rollouts, self.agents, self.envs,
                        [pr.derive_seed(self.seed, 2, self.global_id(p), g) for p in range(self.P)])
        # 2. every pod's learners in one launch, then per-pod fusion
        srcs = [a for a in self.agents for _ in range(self.L)]
        ros = [r for r in self.rollouts for _ in range(self.L)]
        outs = [o for lo in self.learner_out for o in lo]
        seeds = [pr.derive_seed(self.seed, 3, self.global_id(p), l, g) for p in range(self.P) for l in range(self.L)]
        _, stats = pr.ppo_update_learners(srcs, ros, self.cfg, seeds, outs=outs)
        for p in range(self.P):
            pr.fuse_parameters(self.learner_out[p], out=self.agents[p])
        # 3. evaluation scores
        recs = pr.evaluate_pods(self.agents, self.eval_envs,
                                [pr.derive_seed(self.seed, 4, self.global_id(p), g) for p in range(self.P)])
        scores = np.array([rec.mean for rec in recs])
        # 4. leaderboard over every rank's pods (the previous board's entries compete again)
        ids = [self.global_id(p) for p in range(self.P)]
        seqs = [arrival_seq(g, pid, self.world * self.P) for pid in ids]
        if self.comm is not None:
            board, _ = allgather_rank(self.comm, scores, seqs, ids, self.capacity)
        else:
            order = pr.leaderboard_rank(self.ctx, scores, np.asarray(seqs, dtype=np.uint64), self.capacity)
            board = [BoardEntry(float(scores[i]), int(seqs[i]), int(ids[i])) for i in order]
        self.board = board
        # 5. elites (top_k) on every rank, then the next generation's inits
        k = min(self.top_k, len(board))
        for j in range(k):
            pid = board[j].pod_id
            owner = owner_rank(pid, self.P)
            if owner == self.rank:
                self.elites[j].copy_from(self.agents[pid - self.rank * self.P])
            if self.comm is not None:
                broadcast_agent(self.comm, self.elites[j], owner)
        fresh = 0
        for p in range(self.P):
            if k == 0 or self.rng.random() < self.fresh_prob:
                self.agents[p].init_device(int(self.rng.integers(0, 2**63)))  # artifact_init on the device
                fresh += 1
            else:
                self.agents[p].copy_from(self.elites[int(self.rng.integers(0, k))])
                self.agents[p].mutate(int(self.rng.integers(0, 2**63)), self.sigma)
        self.ctx.synchronize()
        self.gen += 1
        self.last_scores = scores
        return {"generation": g, "scores": scores.tolist(), "board": [b.pod_id for b in board], "fresh": fresh,
                "mean_policy_loss": float(np.mean([s.mean_policy_loss for s in stats])),
                "minibatches_per_learner": stats[0].minibatches}
