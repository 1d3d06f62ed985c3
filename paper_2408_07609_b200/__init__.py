"""B200-native nested-grid tsunami time step (arXiv 2408.07609 hot path).

Drop-in for the reference simulator's (``blockswe``) simulation API:
grid/bathymetry setup types, nesting hierarchy, initial displacement,
``Simulation(system, settings, plan).run(n)`` and the max-height /
max-speed / inundation outputs — with every step executed by hand-written
sm_100a CUDA kernels through the C ABI in ``include/tsunami_b200.h``.
"""

from .balance import (B200_MODEL, GPU_REFERENCE_MODEL, CostModel, DecompositionPlan, PlanError,
                      b200_block_weights, b200_phase_weights, concat_plans,
                      phase_balanced_plan, AssignmentPlan, packed_plan, equal_cell_plan, fit_cost_model, minmax_plan,
                      predict_rank_cost, rank_costs, save_cost_model, load_cost_model, measure_block_costs,
                      measure_width_costs, save_width_costs, load_width_costs)
from .grid import (Block, BoundaryConditions, GridLevel, GridStructureError, InitialCondition,
                   NestedGridSystem, SimulationConfig, build_kochi_scaled_config,
                   kochi_block_inventory, kochi_settings, level_abutments,
                   uncovered_side_intervals, validate_system)
from .runner import (PHASE_SEQUENCE, ROUTINES, NumericsError, RunReport, Simulation,
                     SimulationAborted, run_simulation)
from .schedule import build_halo_schedule, build_offset_tables
from . import report  # noqa: E402  (run outputs: rasters, timing CSVs)

__version__ = "0.1.0"

__all__ = [
    "B200_MODEL", "Block", "b200_block_weights", "b200_phase_weights", "phase_balanced_plan", "AssignmentPlan", "packed_plan", "BoundaryConditions", "CostModel", "DecompositionPlan",
    "GPU_REFERENCE_MODEL", "GridLevel", "GridStructureError", "InitialCondition",
    "NestedGridSystem", "NumericsError", "PHASE_SEQUENCE", "PlanError", "ROUTINES", "RunReport",
    "Simulation", "SimulationAborted", "SimulationConfig", "build_halo_schedule",
    "build_kochi_scaled_config", "build_offset_tables", "concat_plans", "equal_cell_plan",
    "fit_cost_model", "kochi_block_inventory", "kochi_settings", "level_abutments",
    "minmax_plan", "predict_rank_cost", "rank_costs", "run_simulation",
    "uncovered_side_intervals", "validate_system", "__version__", "save_cost_model", "load_cost_model",
    "measure_block_costs", "measure_width_costs", "save_width_costs", "load_width_costs",
]
