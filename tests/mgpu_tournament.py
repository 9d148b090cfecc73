"""Multi-GPU tournament check (run under torchrun, one rank per GPU; see
tests/test_gpu_multi.py).  Every rank: device all-gather + ranking of the
pods' (score, seq, pod_id) must equal the reference ordering and agree across
ranks; the elite broadcast must deliver the owner's params/m/v/t."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_05923_b200 import podracer as pr  # noqa: E402
from paper_2112_05923_b200 import tournament as tn  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = pr.Context(local)

    def share(b):
        obj = [b]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    comm = tn.Communicator(ctx, rank, world, share)
    pods, capacity = 8, 10
    for gen in range(4):
        rng = np.random.default_rng(1000 * gen + rank)
        scores = rng.integers(0, 5, pods).astype(np.float64)
        ids = [tn.global_pod_id(rank, i, pods) for i in range(pods)]
        seqs = [tn.arrival_seq(gen, pid, world * pods) for pid in ids]
        board, order = tn.allgather_rank(comm, scores, seqs, ids, capacity)
        gathered = [None] * world
        dist.all_gather_object(gathered, list(zip(scores.tolist(), seqs, ids)))
        cand = [c for part in gathered for c in part]
        ref = tn.rank_candidates_host([c[0] for c in cand], [c[1] for c in cand], capacity)
        assert [b.pod_id for b in board] == [cand[i][2] for i in ref], (rank, gen)
        boards = [None] * world
        dist.all_gather_object(boards, [b.pod_id for b in board])
        assert all(bb == boards[0] for bb in boards)
    # elite broadcast from the owner of the best pod
    agent = pr.Agent.init(ctx, 181, 30, seed=100 + rank)
    flat_rank = agent.flatten_params()
    root = tn.owner_rank(board[0].pod_id, pods)
    tn.broadcast_agent(comm, agent, root)
    got = agent.flatten_params()
    expect = pr.artifact_init(181, 30, 100 + root).astype(np.float32).astype(np.float64)
    assert np.array_equal(got, expect), rank
    if rank != root:
        assert not np.array_equal(flat_rank, got)
    # a real pod population on every rank (configs[3] shape, small): grouped collect, concurrent
    # learners, fusion, evaluation, NCCL all-gather ranking, elite broadcast + mutation
    K = 30
    m = pr.synthetic_market(K, 512, seed=2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    market = pr.MarketData(ctx, m["close"], ind)
    cfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=1, buffer_size=128 * 32)
    pop = tn.PodPopulation(ctx, market, pr.StockConfig(), pods=4, envs_per_pod=128, horizon=32, learners=2,
                           ppo_cfg=cfg, window=(0, 400), eval_episodes=4, eval_window=(300, 340), capacity=5,
                           top_k=3, seed=5, rank=rank, world=world, comm=comm)
    for _ in range(2):
        out = pop.generation()
        boards = [None] * world
        dist.all_gather_object(boards, out["board"])
        assert all(bb == boards[0] for bb in boards), boards
        scores = [None] * world
        dist.all_gather_object(scores, out["scores"])
        flat = [s for part in scores for s in part]
        seqs = [tn.arrival_seq(out["generation"], pid, world * 4) for pid in range(world * 4)]
        assert out["board"] == tn.rank_candidates_host(flat, seqs, 5)
    # the elites are identical on every rank after their broadcasts
    e0 = pop.elites[0].flatten_params()
    sums = [None] * world
    dist.all_gather_object(sums, float(np.sum(e0)))
    assert all(x == sums[0] for x in sums)
    comm.close()
    dist.barrier()
    if rank == 0:
        print("MGPU TOURNAMENT OK", world)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
