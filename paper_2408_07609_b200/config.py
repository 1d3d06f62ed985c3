"""YAML run configs in the reference's format (config.py:35-120).

Top level: ``dt``, optional ``duration``, ``gravity``, ``wet_threshold``,
``manning_n``, ``boundary`` (west/east/south/north: reflective|radiation),
``initial`` (kind rest|gaussian, amplitude, sigma, center), ``rank_budgets``;
then ``levels``: a list of ``{dx, blocks: [{id?, origin, ni, nj,
bathymetry, manning_n?}]}``.  Bathymetry: a number (constant depth),
``{kind: constant, depth}``, ``{kind: slope, d0, gx, gy}`` (depth =
d0 + gx x + gy y at cell centres, global metres), ``{kind: coastal_profile,
y_center, half_extent}`` (the Kochi cubic ramp) or ``{kind: raster, path}``
(``ni x nj`` whitespace-separated values, row-major over x; relative paths
from the config's directory).  Level indices are 1-based in file order;
block ids default to a running counter.
"""

from __future__ import annotations

import os

import numpy as np

from .grid import (DEFAULT_GRAVITY, DEFAULT_MANNING_N, DEFAULT_WET_THRESHOLD, Block, BoundaryConditions,
                   GridLevel, InitialCondition, NestedGridSystem, SimulationConfig, kochi_depth)


class ConfigError(ValueError):
    """The config file is malformed or references missing data."""


def _centres(origin, ni, nj, dx):
    x = origin[0] + (np.arange(ni) + 0.5) * dx
    y = origin[1] + (np.arange(nj) + 0.5) * dx
    return x[:, None], y[None, :]


def bathymetry(spec, origin, ni, nj, dx, base_dir="."):
    """Depth array (ni, nj) of one block's bathymetry section."""
    if isinstance(spec, (int, float)):
        spec = {"kind": "constant", "depth": float(spec)}
    if not isinstance(spec, dict):
        raise ConfigError(f"bathymetry must be a number or a mapping, got {spec!r}")
    kind = spec.get("kind")
    if kind == "constant":
        return np.full((ni, nj), float(spec["depth"]))
    if kind == "slope":
        x, y = _centres(origin, ni, nj, dx)
        return float(spec.get("d0", 0.0)) + float(spec.get("gx", 0.0)) * x + float(spec.get("gy", 0.0)) * y \
            + np.zeros((ni, nj))
    if kind == "coastal_profile":
        _, y = _centres(origin, ni, nj, dx)
        col = kochi_depth(y[0], float(spec["y_center"]), float(spec["half_extent"]))
        return np.broadcast_to(col, (ni, nj))
    if kind == "raster":
        path = spec["path"]
        if not os.path.isabs(path):
            path = os.path.join(base_dir, path)
        flat = np.asarray(np.loadtxt(path), dtype=float).reshape(-1)
        if flat.size != ni * nj:
            raise ConfigError(f"raster {path} holds {flat.size} values, expected {ni}x{nj}")
        return flat.reshape(ni, nj)
    raise ConfigError(f"unknown bathymetry kind {kind!r}")


def load_config(path: str):
    """(NestedGridSystem, SimulationConfig) of a YAML config file."""
    import yaml
    with open(path) as f:
        doc = yaml.safe_load(f)
    if not isinstance(doc, dict):
        raise ConfigError("config root must be a mapping")
    base_dir = os.path.dirname(os.path.abspath(path))
    if "dt" not in doc:
        raise ConfigError("config must set dt")
    init = dict(doc.get("initial", {"kind": "rest"}))
    if "center" in init:
        init["center"] = tuple(float(v) for v in init["center"])
    settings = SimulationConfig(
        dt=float(doc["dt"]),
        total_duration=float(doc.get("duration", 0.0)),
        g=float(doc.get("gravity", DEFAULT_GRAVITY)),
        wet_threshold=float(doc.get("wet_threshold", DEFAULT_WET_THRESHOLD)),
        boundary=BoundaryConditions(**doc.get("boundary", {})),
        initial=InitialCondition(**init),
        rank_budgets=doc.get("rank_budgets"))
    default_n = float(doc.get("manning_n", DEFAULT_MANNING_N))
    system = NestedGridSystem()
    next_id = 1
    for k, lvl_doc in enumerate(doc.get("levels", [])):
        level = GridLevel(level_index=k + 1, dx=float(lvl_doc["dx"]))
        for blk in lvl_doc.get("blocks", []):
            origin = tuple(float(v) for v in blk["origin"])
            ni, nj = int(blk["ni"]), int(blk["nj"])
            h = bathymetry(blk["bathymetry"], origin, ni, nj, level.dx, base_dir)
            block_id = int(blk.get("id", next_id))
            next_id = max(next_id, block_id) + 1
            level.blocks.append(Block(block_id=block_id, origin=origin, ni=ni, nj=nj, h=h,
                                      manning_n=float(blk.get("manning_n", default_n))))
        system.levels.append(level)
    if not system.levels:
        raise ConfigError("config defines no grid levels")
    return system, settings
