"""Multi-process CPU tests of the queue-sharding layer (world_size 2, gloo backend): shards
partition the global queue and keep the mix; the counter all-gather sums to the submitted
totals; the global throughput uses max t_end - min t_start."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import kl_inputs as G
from paper_1303_5164_b200 import dist as KD


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gq = G.queue("ALL", 32 * world, order="round_robin")
    mine = KD.shard(gq, rank, world)
    # emulate this rank's completion counters as the kernels would write them
    c = torch.tensor([len(mine), 100 * len(mine), 1000 + rank, 5000 + 10 * rank,
                      sum(i + 1 for i, e in enumerate(gq) if i % world == rank), rank, world, 3], dtype=torch.int64)
    g = KD.allgather_counters(c)
    s = KD.global_summary(g)
    q.put((rank, [e["kind"] for e in mine], s))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_and_allgather_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    gq = [e["kind"] for e in G.queue("ALL", 64, order="round_robin")]
    assert sorted(res[0][1] + res[1][1]) == sorted(gq)
    for r in res:
        assert {k: r[1].count(k) for k in set(r[1])} == {k: 4 for k in G.MIXES["ALL"]}   # mix kept
        s = r[2]
        assert s["kernels_done"] == 64 and s["blocks_done"] == 6400
        assert s["checksum"] == sum(range(1, 65))
        assert s["span_ns"] == 5010 - 1000


def test_lpt_shard_balances():
    q = [{"kind": k, "cost": c} for k, c in zip("abcdefgh", [9, 1, 1, 1, 5, 4, 2, 1])]
    parts = [KD.shard(q, r, 2, mode="lpt", cost=lambda e: e["cost"]) for r in range(2)]
    loads = [sum(e["cost"] for e in p) for p in parts]
    assert sorted(sum(parts, []), key=lambda e: e["kind"]) == q
    assert abs(loads[0] - loads[1]) <= 1
