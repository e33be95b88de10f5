"""paper_2404_01931_b200 — B200-native (sm_100a) PIC/FLIP timestep.

Drop-in for the simulation path of the reference package ``flipsim``
(arXiv 2404.01931): SceneSpec / make_scene / step / SimState accessors and
the kernel-backend plugin API, executed by hand-written CUDA kernels in
``libflipb200.so`` (C ABI: include/flipb200.h).  Importing fails if the
library is not built; there is no CPU fallback.
"""

from . import _kernels
from ._kernels import backend_name, set_backend, set_workers
from ._lib import LIB_PATH, device_count
from .binning import SpaceHash
from .errors import (ConfigError, FlipsimError, SingularSystemError, SolverBreakdownError,
                     SolverError)
from .grid import AIR, FLUID, SOLID, GridDims, MacGrid, cell_coords, flat_index
from .particles import MAX_PER_CELL, MIN_PER_CELL, ParticleSet, SeedRegion
from .pressure import SolveResult, solve
from .sim import (SCENE_NAMES, SceneSpec, SimState, StageTimings, StepReport, divergence_field,
                  energy_floor, make_scene, run_stages, scene_regions, step, total_energy)

__version__ = "0.1.0"
