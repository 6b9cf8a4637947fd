"""B200-native backend for the hexmc per-sample supercell solve (arXiv 1611.09784).

Same public names as the reference package (pkg/src/hexmc/__init__.py:5-29) for the hot path:
models, geometry, sampling, BZ grids, band solves, IDOS, level moments and the Engine whose
`evaluate_masks` batch seam runs on libhx.so (hand-written sm_100a CUDA, C-ABI in include/hx.h).
"""

from .engine import SLMC_STREAM_OFFSET, Engine, ExhaustiveResult, LevelSampleSet, TaskError
from .estimators import (LevelPlan, LevelStats, MlmcEstimate, combine_levels, control_variate_sample, level_moments,
                         mean_and_variance, window_mask)
from .geometry import LatticeSpec, PartitionMap, Supercell, build_supercell, honeycomb, partition_quarters
from .idos import EnergyGrid, IdosCurve, SmoothingSpec, dos_by_differentiation, idos, idos_sharp, smoothing_g
from .models import (BlochOperatorPair, CompiledCell, GrapheneNNModel, MultiOrbitalModel, assemble_bloch,
                     compile_cell, hermiticity_check, load_coupling_table)
from .sampling import DefectConfiguration, SeedSpec, enumerate_configs, restrict, sample_defects
from .solver import BandGrid, BzGrid, SolverError, estimate_solve_cost, make_bz_grid, solve_bands

__version__ = "0.1.0"
