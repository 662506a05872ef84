"""B200-native backend for the Celerity/SYnergy-style distributed data-parallel
model of arXiv 2505.06022 -- a drop-in for the reference ``clusterq`` API
(reference: pkg/src/clusterq/__init__.py:4-59).

The host side (this package) keeps the reference's queue/submit, range
mappers, task graph, command planner and SYnergy energy selection, bit-exact.
Execution -- the layer the reference simulates with a per-cell Python loop
(pkg/src/clusterq/simulator.py:101-224) -- is replaced by ``executor.run``,
which drives hand-written sm_100a kernels, NVLink/NCCL transfers and NVML
energy counters through the ``libcq`` C-ABI (include/cq.h) via ctypes.
There is no CPU execution path: without the native library ``run`` raises.
"""

from .energy import (
    DeviceModel,
    EnergyReport,
    EnergyTarget,
    account_energy,
    resolve_target,
    select_frequency,
)
from .errors import (
    ClusterqError,
    DimensionError,
    EvalError,
    KernelNameError,
    KernelSyntaxError,
    MapperViolationError,
    NativeError,
    ScenarioError,
    UninitializedReadError,
    ValidationError,
)
from .graph import TaskGraph
from .kernel import format_kernel, parse_kernel
from .model import (
    Accessor,
    AccessMode,
    All,
    Buffer,
    BufferInit,
    Fixed,
    NativeKernel,
    Neighborhood,
    OneToOne,
    Slice,
    Task,
)
from .region import Box, Region
from .scheduler import (
    AwaitPushCommand,
    ExecuteCommand,
    Plan,
    PushCommand,
    RegionMapTable,
    export_command_graph,
    generate_commands,
    split_task,
)

__version__ = "0.1.0"


def __getattr__(name):
    # The executor pulls in the ctypes binding lazily so that planning-only
    # users (and the CPU test suite) never need the native library.
    if name in ("run", "run_batch", "RunResult", "TraceEvent", "LinkModel", "trace_to_chrome"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)
