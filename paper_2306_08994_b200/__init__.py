"""B200-native multifrontal factor/solve behind the `tracefront` API.

Mirrors the reference package's public names (tracefront/__init__.py:10-37)
for the hot path: FEM fronts -> elimination tree -> symbolic plan -> Foata
(level) schedule -> GPU factorization -> solve.  The numeric path is
hand-written sm_100a CUDA in libtfb200.so; nothing falls back to the CPU.
"""

from .errors import (
    ContractViolationError,
    CycleError,
    EmptyInputError,
    InvalidGeometryError,
    SymbolicSingularityError,
    TracefrontError,
    UnsupportedDegreeError,
    ZeroPivotError,
)
from .fem import (
    ElementSystem,
    Front,
    FrontSet,
    GlobalSystem,
    Mesh,
    TensorMesh,
    assemble_system,
    element_mass_matrix,
    generate_fronts,
)
from .tree import EliminationTree, TreeNode, build_elimination_tree, join_fronts, sort_fronts
from .symbolic import EliminationPlan, NodeReorder, PivotStep, symbolic_eliminate
from .tasks import (DagReport, DependencyGraph, Task, build_dependency_edges, build_task_graph,
                    enumerate_tasks, validate_dag)
from .schedule import (AtomicFoataSchedule, FoataSchedule, TaskKind, compute_atomic_fnf,
                       compute_fnf, schedule_stats, schedule_stats_csv)
from .engine import (
    ExecState,
    FactorResult,
    compile_execution,
    factor_and_solve,
    factorize,
    init_state,
    run_concurrent,
    run_sequential,
    solve,
)

__version__ = "0.1.0"
