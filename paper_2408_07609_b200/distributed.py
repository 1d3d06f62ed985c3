"""Multi-GPU plumbing: one process per GPU.

Blocks are assigned to GPUs as consecutive runs of the level-ordered block
list, exactly the reference's DecompositionPlan semantics (balance.py:
102-144): plan rank r == GPU r.  Each process owns its blocks' arena on its
GPU; the exchange kernels of the owning (sending) GPU store straight into
the receiving GPU's arena over NVLink, which every process maps with CUDA
IPC.  torch.distributed is only the setup/teardown plumbing: it carries the
IPC handle blobs, reduces the first error over ranks and gathers outputs —
nothing on the per-step path.

The helpers take plain callables so the coordination logic is testable on
CPU with the gloo backend (tests/test_distributed.py).
"""

from __future__ import annotations

import os


def dist_context(group=None):
    """(rank, world_size, local_rank) of this process; (0, 1, 0) when
    torch.distributed is not initialised."""
    try:
        import torch.distributed as dist
    except ImportError:                                   # pragma: no cover
        return 0, 1, 0
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1, int(os.environ.get("LOCAL_RANK", "0"))
    return (dist.get_rank(group), dist.get_world_size(group),
            int(os.environ.get("LOCAL_RANK", str(dist.get_rank(group)))))


def owners_from_plan(system, plan, world: int):
    """Owner rank of every block in global order; the plan must have exactly
    one rank per process."""
    if plan.n_ranks != world:
        raise ValueError(f"plan has {plan.n_ranks} ranks but {world} processes (one per GPU)")
    return [plan.rank_of(k) for k in range(system.n_blocks)]


def all_gather_bytes(blob: bytes, group=None) -> list:
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def exchange_peer_handles(export_fn, import_fn, rank: int, world: int, group=None):
    """Every rank exports its IPC blob; every rank imports all peers'."""
    blobs = all_gather_bytes(export_fn(), group)
    for p in range(world):
        if p != rank:
            import_fn(p, blobs[p])
    return blobs


_FLAGS = {}


def first_error(local, group=None):
    """The reference's first failure over ranks: the minimum of the local
    (block order, what, i, j) keys, or None.  A numerics failure ranks ahead
    of a runtime failure (block order -1, e.g. a peer that stopped at a phase
    barrier because of it).  All ranks get the same answer."""
    import torch
    import torch.distributed as dist
    # the common case (no rank failed) costs one small all-reduce on a
    # persistent flag instead of the pickled all-gather (~1 ms over NCCL,
    # inside every run() call)
    dev = (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
           else torch.device("cpu"))
    key = (id(group), str(dev))
    flag = _FLAGS.get(key)
    if flag is None:
        flag = _FLAGS[key] = torch.zeros(1, dtype=torch.int32, device=dev)
    flag.fill_(0 if local is None else 1)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if int(flag.item()) == 0:
        return None
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local, group=group)
    keys = [k for k in out if k is not None]
    return min(keys, key=lambda k: (k[0] < 0, k)) if keys else None


def max_over_ranks(value: float, group=None) -> float:
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, float(value), group=group)
    return max(out)


def gather_fields(local: dict, root: int = 0, group=None):
    """Merge per-rank {block_id: payload} dicts on ``root`` (None elsewhere)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = [None] * world if dist.get_rank(group) == root else None
    dist.gather_object(local, out, dst=root, group=group)
    if out is None:
        return None
    merged = {}
    for part in out:
        merged.update(part)
    return merged
