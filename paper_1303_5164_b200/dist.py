"""Multi-GPU layer ("extended to multiple GPUs with a workload
dispatcher"): one process per GPU, each with its own Kernelet context, a static shard of the
global queue, and one collective -- an all-gather of the per-GPU completion counters
(kl_counters, int64[8]) over NCCL (gloo on CPU for tests).  No kernel data crosses GPUs."""
from __future__ import annotations

import torch
import torch.distributed as dist

COUNTER_FIELDS = ["kernels_done", "blocks_done", "t_start_ns", "t_end_ns", "checksum", "rank", "world", "phases"]


def shard(queue: list, rank: int, world: int, mode: str = "round_robin", cost=None) -> list:
    """This rank's part of the global queue.
    round_robin: the j-th arrival of each kind goes to rank (j + kind offset) mod world, so every
                 shard keeps the kind proportions of the mix (and so its pairing opportunities);
                 arrival order is kept inside each shard.
    lpt:         longest-predicted-time-first onto the least loaded rank (cost(entry) -> float),
                 arrival order kept inside each shard."""
    if world <= 1:
        return list(queue)
    if mode == "round_robin":
        seen, offs, out = {}, {}, []
        for e in queue:
            k = e["kind"] if isinstance(e, dict) else e
            if k not in offs:
                offs[k] = len(offs) % world
            j = seen.get(k, 0)
            seen[k] = j + 1
            if (j + offs[k]) % world == rank:
                out.append(e)
        return out
    if mode == "lpt":
        assert cost is not None
        order = sorted(range(len(queue)), key=lambda i: (-cost(queue[i]), i))
        load = [0.0] * world
        owner = [0] * len(queue)
        for i in order:
            r = min(range(world), key=lambda x: (load[x], x))
            owner[i] = r
            load[r] += cost(queue[i])
        return [e for i, e in enumerate(queue) if owner[i] == rank]
    raise ValueError(mode)


def allgather_counters(counters: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather the int64[8] counter block of every rank -> (world, 8) tensor on the same
    device (NCCL reads the device buffer the kernels wrote)."""
    world = dist.get_world_size(group)
    out = torch.empty(world * counters.numel(), dtype=counters.dtype, device=counters.device)
    dist.all_gather_into_tensor(out, counters.contiguous(), group=group)
    return out.view(world, counters.numel())


def global_summary(gathered: torch.Tensor) -> dict:
    """Whole-job completion and throughput from the gathered counters: total kernels over
    (max t_end - min t_start) on the shared host clock."""
    g = gathered.cpu().tolist()
    kern = sum(r[0] for r in g)
    t0 = min(r[2] for r in g)
    t1 = max(r[3] for r in g)
    return {"kernels_done": kern, "blocks_done": sum(r[1] for r in g), "checksum": sum(r[4] for r in g),
            "span_ns": t1 - t0, "kernels_per_s": kern / ((t1 - t0) / 1e9) if t1 > t0 else 0.0,
            "per_rank": [dict(zip(COUNTER_FIELDS, r)) for r in g]}
