"""The reference's own objects work unchanged: a
blockswe NestedGridSystem / SimulationConfig / DecompositionPlan fed to the
product's builders gives exactly what the product's own types give —
exchange tables, domain edges, host arrays and the whole C-ABI descriptor
(CPU only: the library is loaded, no device call).  Needs the reference
under /root/reference (the build container); skipped elsewhere."""

import ctypes
import os
import sys

import numpy as np
import pytest

import systems
from conftest import REFERENCE_SRC

pytestmark = pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="needs the reference sources")

CASES = systems.SMALL + ("kochi",)


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REFERENCE_SRC)
    import blockswe
    import blockswe.grid
    return blockswe


def _pair(product, ref, name):
    if name == "kochi":
        return systems.kochi(ref.grid, 0.001)[:2], systems.kochi(product, 0.001)[:2]
    return systems.make(ref.grid, name)[:2], systems.make(product, name)[:2]


def _struct_rows(arr, n):
    return [tuple(getattr(arr[k], f) for f, _ in type(arr[k])._fields_) for k in range(n)]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("nr", (1, 3))
def test_reference_objects_drive_the_product(product, ref, name, nr):
    from paper_2408_07609_b200 import distributed as D
    from paper_2408_07609_b200 import schedule as S
    from paper_2408_07609_b200.runner import build_descriptor, host_block_arrays
    (rsys, rset), (psys, pset) = _pair(product, ref, name)
    assert type(rsys).__module__.startswith("blockswe")
    nr = min(nr, rsys.n_blocks)
    cells = [b.cell_count for _, b in rsys.all_blocks()]
    rplan = ref.equal_cell_plan(cells, nr)                   # the reference's DecompositionPlan
    pplan = product.equal_cell_plan(cells, nr)
    assert [rplan.rank_of(k) for k in range(rplan.n_blocks)] == [pplan.rank_of(k) for k in range(pplan.n_blocks)]
    rank_of = {b.block_id: rplan.rank_of(k) for k, (_, b) in enumerate(rsys.all_blocks())}

    rh, ph = S.build_halo_schedule(rsys, rank_of), S.build_halo_schedule(psys, rank_of)
    assert repr(rh.entries) == repr(ph.entries) and rh.lengths == ph.lengths
    rt, pt = S.build_offset_tables(rsys, rank_of), S.build_offset_tables(psys, rank_of)
    assert repr(rt.links) == repr(pt.links) and rt.buffer_len == pt.buffer_len
    re_, pe_ = S.domain_edges(rsys, rset, rank_of), S.domain_edges(psys, pset, rank_of)
    assert re_ == pe_

    ra, pa = host_block_arrays(rsys, rset), host_block_arrays(psys, pset)
    assert ra.keys() == pa.keys()
    for bid in ra:
        for x, y in zip(ra[bid], pa[bid]):
            assert (x is None) == (y is None)
            if x is not None:
                assert np.array_equal(x.view(np.uint64), y.view(np.uint64))

    owner = D.owners_from_plan(rsys, rplan, nr) if nr > 1 else [0] * rsys.n_blocks
    rd, rkeep = build_descriptor(rsys, rset, owner, rh, rt, re_, rank=0, world=nr)
    pd, pkeep = build_descriptor(psys, pset, owner, ph, pt, pe_, rank=0, world=nr)
    for f in ("n_blocks", "dt", "gravity", "wet_threshold", "n_halo", "n_restrict", "n_prolong", "n_edges",
              "rank", "n_ranks"):
        assert getattr(rd, f) == getattr(pd, f), f
    for k in range(rd.n_blocks):
        a, b = rd.blocks[k], pd.blocks[k]
        for f in ("block_id", "ni", "nj", "owner", "level", "dx", "manning"):
            assert getattr(a, f) == getattr(b, f), (k, f)
    for arr, n in (("halo", rd.n_halo), ("restrict_segs", rd.n_restrict), ("prolong_segs", rd.n_prolong),
                   ("edges", rd.n_edges)):
        assert _struct_rows(getattr(rd, arr), n) == _struct_rows(getattr(pd, arr), n), arr


def test_reference_config_file_loads_into_the_product(product, ref):
    """A YAML config read by the reference's loader (config.py:73-121) gives
    the same host arrays as the product's loader on the same file."""
    from paper_2408_07609_b200.config import load_config
    from paper_2408_07609_b200.runner import host_block_arrays
    path = os.path.join(os.path.dirname(__file__), "golden", "configs", "cfg2.yaml")
    rsys, rset = ref.load_config(path)
    psys, pset = load_config(path)
    ra, pa = host_block_arrays(rsys, rset), host_block_arrays(psys, pset)
    for bid in ra:
        for x, y in zip(ra[bid], pa[bid]):
            if x is not None:
                assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
