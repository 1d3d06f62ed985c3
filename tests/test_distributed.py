"""Multi-process host logic of the multi-GPU path, on CPU with gloo
(world size 2): IPC-blob exchange, first-error agreement, max-over-ranks
timing, output gathering and plan -> owner mapping.  The device side (peer
stores, NVLink barriers) is covered by tools/mgpu_check.py on >= 2 GPUs."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2408_07609_b200 import distributed as D


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = D.dist_context()
        imported = []
        blobs = D.exchange_peer_handles(lambda: bytes([r]) * 8, lambda p, b: imported.append((p, b)), r, w)
        assert [b[0] for b in blobs] == list(range(w))
        assert imported == [(p, bytes([p]) * 8) for p in range(w) if p != r]
        # rank 1 fails in block 5 at (2, 3); rank 0 has no error -> both see it
        first = D.first_error((5, 1, 2, 3) if r == 1 else None)
        assert first == (5, 1, 2, 3)
        first = D.first_error((7, 0, 0, 0) if r == 0 else (5, 2, 1, 1))
        assert first == (5, 2, 1, 1)
        assert D.first_error(None) is None
        # a runtime failure (peer stopped at a barrier) never masks a
        # numerics failure of another rank
        first = D.first_error((-1, 9, 0, 0, "barrier") if r == 0 else (3, 0, 4, 4))
        assert first == (3, 0, 4, 4)
        assert D.max_over_ranks(0.5 + r) == 0.5 + (w - 1)
        merged = D.gather_fields({10 + r: r}, root=0)
        if r == 0:
            assert merged == {10 + k: k for k in range(w)}
        else:
            assert merged is None
        q.put((r, "ok"))
    except Exception as exc:          # surfaced by the parent
        q.put((r, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_rank_coordination_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}


def test_owners_from_plan():
    import paper_2408_07609_b200 as P
    system = P.build_kochi_scaled_config(0.001)
    cells = [b.cell_count for _, b in system.all_blocks()]
    plan = P.minmax_plan(cells, 4)
    owners = D.owners_from_plan(system, plan, 4)
    assert owners == sorted(owners) and set(owners) == {0, 1, 2, 3}
    with pytest.raises(ValueError):
        D.owners_from_plan(system, plan, 2)
