"""B200-native LASGD parameter-synchronisation path (arXiv 2203.13085).

Drop-in for the reference package's sync path (``lasgd.params``,
``lasgd.collective``, ``lasgd.optimizer``, ``lasgd.problems.lr_at``): the same
names and argument order, device buffers instead of host vectors, fused
sm_100a kernels behind a C ABI (include/lasgd_sync.h) instead of numpy.

Importing this package loads ``_lib/liblasgd_sync.so`` eagerly and raises
``ImportError`` if it is missing — there is no CPU fallback.
"""

from . import _native

_native.lib()  # fail loudly at import time when the CUDA library is absent

from ._native import CollectiveFailure, DimensionMismatchError, NonFiniteError, TransportFault  # noqa: E402
from .collective import (  # noqa: E402
    AllReduceOutcome,
    CollectiveHandle,
    CudaLoopbackTransport,
    CudaP2PTransport,
    P2PCommunicator,
    RingSchedule,
    RingStep,
    Status,
    all_reduce_average,
    bytes_per_node,
    execute_allreduce,
    poll,
    ring_schedule,
)
from .engine import BucketedSGDARWorker, LASGDWorker, SGDARWorker, SyncGraph  # noqa: E402
from .torch_optim import LASGD  # noqa: E402
from .graphs import GraphedStep  # noqa: E402
from .flat import FlatParams  # noqa: E402
from .optimizer import (  # noqa: E402
    easgd_round_robin_exchange,
    elastic_center_step,
    elastic_local_step,
    HyperParamError,
    HyperParams,
    ModelDivergenceError,
    NodeState,
    SgdConfig,
    TickAction,
    lasgd_finalize_round,
    lasgd_node_tick,
    sgd_local_step,
    sync_allreduce_sgd_round,
)
from .params import ChunkSpec, as_device_vector, blend, mean_of_vectors, partition_chunks, require_same_dim  # noqa: E402
from .problems import LrSchedule, lr_at  # noqa: E402

__all__ = [
    "BucketedSGDARWorker", "ChunkSpec", "LASGD", "CollectiveFailure", "CollectiveHandle", "CudaLoopbackTransport", "CudaP2PTransport",
    "DimensionMismatchError", "FlatParams", "GraphedStep", "HyperParamError", "HyperParams", "LASGDWorker", "LrSchedule", "SyncGraph", "ModelDivergenceError",
    "NodeState", "NonFiniteError", "P2PCommunicator", "RingSchedule", "RingStep", "SGDARWorker", "SgdConfig", "Status", "TickAction", "TransportFault",
    "AllReduceOutcome", "all_reduce_average", "as_device_vector", "execute_allreduce", "blend", "bytes_per_node", "easgd_round_robin_exchange",
    "elastic_center_step", "elastic_local_step", "mean_of_vectors", "lasgd_finalize_round", "lasgd_node_tick",
    "lr_at", "partition_chunks", "poll", "require_same_dim", "ring_schedule", "sgd_local_step", "sync_allreduce_sgd_round",
]
