"""YAML configs (the reference's format) and the command line."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import systems
from conftest import GOLDEN

CONFIGS = os.path.join(GOLDEN, "configs")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ("cfg1", "cfg2"))
def test_load_config_matches_fixture_and_reference_digests(product, name):
    from paper_2408_07609_b200.config import load_config
    system, settings = load_config(os.path.join(CONFIGS, f"{name}.yaml"))
    ref_system, ref_settings, _ = systems.make(product, name)
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        digests = json.load(f)[name]
    assert [b.block_id for _, b in system.all_blocks()] == [b.block_id for _, b in ref_system.all_blocks()]
    for (lvl, b), (rl, rb) in zip(system.all_blocks(), ref_system.all_blocks()):
        assert lvl.dx == rl.dx and (b.ni, b.nj, tuple(b.origin)) == (rb.ni, rb.nj, tuple(rb.origin))
        assert np.array_equal(b.h, rb.h)
        assert systems.digest(b.h) == digests["h"][str(b.block_id)]      # the reference's own bathymetry
        assert b.manning_n == rb.manning_n
    for attr in ("dt", "total_duration", "g", "wet_threshold"):
        assert getattr(settings, attr) == getattr(ref_settings, attr)
    for side in ("west", "east", "south", "north"):
        assert getattr(settings.boundary, side) == getattr(ref_settings.boundary, side)
    for attr in ("kind", "amplitude", "sigma", "center"):
        assert getattr(settings.initial, attr) == getattr(ref_settings.initial, attr)


def test_config_errors(product, tmp_path):
    from paper_2408_07609_b200.config import ConfigError, load_config
    p = tmp_path / "bad.yaml"
    p.write_text("levels: []\n")
    with pytest.raises(ConfigError):
        load_config(str(p))
    p.write_text("dt: 0.2\nlevels: []\n")
    with pytest.raises(ConfigError):
        load_config(str(p))
    p.write_text("dt: 0.2\nlevels: [{dx: 10.0, blocks: [{origin: [0, 0], ni: 2, nj: 2, "
                 "bathymetry: {kind: nope}}]}]\n")
    with pytest.raises(ConfigError):
        load_config(str(p))
