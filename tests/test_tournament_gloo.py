"""CPU, world_size 2 (gloo): the tournament's cross-rank bookkeeping.

Each rank owns a pod population; scores are all-gathered and every rank must
derive the identical board -- the order sequential leaderboard_update
insertion gives (tournament.hpp:104-119, checked against the C oracle) --
and agree on which rank owns each elite (the broadcast root)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, pods, capacity, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2112_05923_b200 import tournament as tn
    results = []
    for gen in range(3):
        rng = np.random.default_rng(100 * gen + rank)
        scores = rng.integers(0, 4, pods).astype(float).tolist()  # heavy ties across ranks
        ids = [tn.global_pod_id(rank, i, pods) for i in range(pods)]
        seqs = [tn.arrival_seq(gen, pid, world * pods) for pid in ids]
        gathered = [None] * world
        dist.all_gather_object(gathered, list(zip(scores, seqs, ids)))
        cand = [c for part in gathered for c in part]
        order = tn.rank_candidates_host([c[0] for c in cand], [c[1] for c in cand], capacity)
        board = [cand[i] for i in order]
        owners = [tn.owner_rank(c[2], pods) for c in board]
        results.append((board, owners, cand))
    q.put((rank, results))
    dist.destroy_process_group()


def test_two_rank_board_agreement(orc):
    from oracle_bind import I64, U64, ptr
    world, pods, capacity = 2, 4, 5
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pods, capacity, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1]  # identical board and elite owners on every rank
    for board, owners, cand in out[0]:
        # equals sequential insertion of ALL candidates in arrival (seq) order through the
        # oracle's leaderboard_update (which is pinned to the reference's)
        all_cands = sorted(cand, key=lambda c: c[1])
        bs = np.zeros(capacity); bq = np.zeros(capacity, dtype=np.uint64); bi = np.zeros(capacity, dtype=np.int64)
        size = C.c_size_t(0); seq = C.c_uint64(0)
        for s, _, pid in all_cands:
            orc.orc_leaderboard_update(ptr(bs), ptr(bq, U64), ptr(bi, I64), C.byref(size), capacity, C.byref(seq),
                                       float(s), int(pid))
        assert [c[2] for c in board] == list(bi[:size.value])
        assert owners == [c[2] // pods for c in board]
