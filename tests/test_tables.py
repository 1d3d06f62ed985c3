"""Exchange tables equal the reference's own (tests/golden/tables.json,
dumped from blockswe.build_halo_schedule / build_offset_tables /
uncovered_side_intervals / equal_cell_plan on every fixture system, Kochi-0.001
and Kochi-1.0 at 1/2/4/8 ranks).  Both the product's builders and the
oracle's restatement are checked."""

import json
import os

import numpy as np
import pytest

import systems
from conftest import GOLDEN

with open(os.path.join(GOLDEN, "tables.json")) as f:
    TABLES = json.load(f)


def _system(P, key):
    name = key.split("/")[0]
    if name == "kochi1":
        s, st, _ = systems.kochi(P, 1.0)
        return s, st
    s, st, _ = systems.make(P, name)
    return s, st


def _rank_of(P, system, nr):
    plan = P.equal_cell_plan([b.cell_count for _, b in system.all_blocks()], nr)
    return plan, {b.block_id: plan.rank_of(k) for k, (_, b) in enumerate(system.all_blocks())}


@pytest.mark.parametrize("key", sorted(TABLES))
def test_product_tables_equal_reference(product, key):
    want = TABLES[key]
    system, settings = _system(product, key)
    plan, rank_of = _rank_of(product, system, want["n_ranks"])
    assert list(plan.separators) == want["separators"]
    from paper_2408_07609_b200 import schedule as S
    halo = S.build_halo_schedule(system, rank_of)
    got = [[s, r, [[e.block_id, e.peer_id, e.side, *e.send_span, *e.recv_span, e.eta_offset,
                    e.flux_offset] for e in halo.entries[(s, r)]]] for (s, r) in sorted(halo.entries)]
    assert got == want["halo"]
    assert sorted([s, r, p, n] for (s, r, p), n in halo.lengths.items()) == want["halo_lengths"]
    tabs = S.build_offset_tables(system, rank_of)
    got = [[ln.parent_block, ln.child_block,
            [[g.side, *g.child_span, g.ring_start, g.parent_line, *g.parent_span, g.offset, g.length]
             for g in ln.eta_segments],
            [[g.side, *g.child_span, g.child_face_line, g.parent_face_line, *g.parent_span, g.offset,
              g.length] for g in ln.flux_segments]] for ln in tabs.links]
    assert got == want["links"]
    got = [[*k, [[ln.parent_block, ln.child_block] for ln in tabs.pair_links[k]]]
           for k in sorted(tabs.pair_links)]
    assert got == want["pair_links"]
    assert sorted([s, r, p, n] for (s, r, p), n in tabs.buffer_len.items()) == want["buffer_len"]
    edges = S.domain_edges(system, settings, rank_of)
    got = [[r, bid, side, iv[0], iv[1], kind] for r in sorted(edges) for (bid, side, iv, kind) in edges[r]]
    assert sorted(got) == sorted(want["edges"])


@pytest.mark.parametrize("key", sorted(k for k in TABLES if not k.startswith("kochi1")))
def test_oracle_tables_equal_reference(oracle_mod, product, key):
    want = TABLES[key]
    system, settings = _system(product, key)
    _, rank_of = _rank_of(product, system, want["n_ranks"])
    ents = oracle_mod.halo_entries(system, rank_of)
    got = {}
    for (s, r), lst in ents.items():
        got[(s, r)] = [[e.sender, e.receiver, e.side, *e.send_span, *e.recv_span] for e in lst]
    for s, r, lst in want["halo"]:
        assert got[(s, r)] == [e[:7] for e in lst]
    links = oracle_mod.intergrid_segments(system)
    assert [[p, c, [list(x) for x in eta], [list(x) for x in flux]] for (p, c, eta, flux) in links] == \
        [[p, c, [e[:7] for e in eta], [f[:7] for f in flux]] for (p, c, eta, flux) in want["links"]]


def test_kochi_inventory_matches_paper(product):
    s = product.build_kochi_scaled_config(1.0)
    assert s.cell_count == 47_211_444          # PAPER.md Table I
    assert [len(l.blocks) for l in s.levels] == [1, 3, 9, 11, 60]
    assert [l.dx for l in s.levels] == [810.0, 270.0, 90.0, 30.0, 10.0]
    assert [l.blocks[0].nj for l in s.levels] == [90, 36, 24, 48, 60]


def test_misaligned_interface_raises(product):
    T = product
    system = T.NestedGridSystem(levels=[
        T.GridLevel(1, 9.0, [systems.flat_block(T, 1, (0.0, 0.0), 6, 6, 8.0)]),
        T.GridLevel(2, 3.0, [systems.flat_block(T, 2, (3.0, 3.0), 8, 8, 8.0)])])
    with pytest.raises(T.GridStructureError):
        T.build_offset_tables(system)
