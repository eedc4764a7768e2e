"""MONeT (arXiv 2010.14501) on B200: budgeted, recompute-scheduled training.

The public surface mirrors the reference planner ``remsched``
(pkg/src/remsched/__init__.py:5-94): graph and catalog documents in, a byte
budget in, a schedule out, and the schedule's exact byte ledger.  On top of
that contract this package *executes* schedules on a B200 with hand-written
sm_100a kernels (``execute`` / ``Runtime``), traces torch models into graph
documents (``trace_graph``) and profiles kernel variants into catalogs
(``profile``).
"""

__version__ = "0.1.0"

from .units import FormatError, format_cost, parse_bytes, parse_cost
from .graph import DependencySets, Graph, compute_dependency_sets, graph_to_doc, load_graph
from .costmodel import (ABLATION_MODES, Catalog, apply_ablation, bundled_fixture,
                        catalog_to_doc, generate_synthetic, load_catalog, resnet_toy)
from .memmodel import MemModel, schedule_cost
from .bound import check_schedule
from .schedule import (Schedule, SimulationError, StagePlan, Trace, checkpoint_heuristic,
                       decode, schedule_from_doc, schedule_to_doc, simulate,
                       store_everything_schedule, trace_report, validate)

from .ilp import (Model, assignment_from_schedule, build_model, evaluate_assignment,
                  export_lp, export_lp_string)
from .solver import SolveResult, lower_bound, propagate, solve
from .enumerate import ORACLE_DEFAULTS, OracleResult, cross_check, enumerate_schedules
from . import enumerate as oracle  # the reference names this module `oracle` (oracle.py)
from . import ilp, solver  # noqa: E402  (module attributes, as in remsched/__init__.py)


def __getattr__(name):
    # the GPU executor is imported lazily so the planner works without CUDA
    if name in ("execute", "Runtime", "BudgetExceeded", "ExecResult"):
        from . import engine
        return getattr(engine, name)
    if name in ("trace_graph", "build_network"):
        from . import tracer
        return getattr(tracer, name)
    if name == "profile":
        from . import profiler
        return profiler.profile
    raise AttributeError(name)
