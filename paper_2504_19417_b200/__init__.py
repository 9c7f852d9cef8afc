"""B200-native VecKM_flow normal-flow estimator (arXiv 2504.19417).

Drop-in for the reference `evflow` estimator path:

    from paper_2504_19417_b200 import NormalFlowRegressor
    flows = NormalFlowRegressor(width=640, height=480, weights="head.vkmw").predict(X)

`X` is an (n, 3) array of [t, x, y]; the result is (n, 2) float64 [n_x, n_y].
`paper_2504_19417_b200.stream` loads EVN1/CSV event files, slices streams like
the reference's `slice_stream`, and `NormalFlowRegressor.predict_stream` runs
every window through one pipelined batch.
`paper_2504_19417_b200.bindings` mirrors the reference's array-in/array-out
`evflow_bindings` (encode / predict / load_config_preset).
Per-event work runs in hand-written sm_100a kernels behind the C-ABI in
include/veckm.h (libveckm.so); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .engine import FlowEngine
from .errors import (
    DimensionMismatchError,
    EmptyNeighborhoodError,
    EventParseError,
    EvflowError,
    GeometryError,
)
from .estimators import LocalEventEncoder, NormalFlowRegressor
from .training import TrainConfig, TrainingDivergedError, train_head
from .stream import CameraGeometry, EventSlice, EventStream
from .validation import block_from_array, check_event_array, check_events, check_flow_array, slice_from_array
from .weights import (
    Bases,
    MlpWeights,
    generate_bases,
    init_weights,
    load_weights,
    save_weights,
    standard_normals,
)

__all__ = [
    "FlowEngine", "NormalFlowRegressor", "LocalEventEncoder", "Bases", "MlpWeights", "generate_bases",
    "init_weights", "load_weights", "save_weights", "standard_normals", "check_event_array",
    "check_flow_array", "slice_from_array", "block_from_array", "check_events", "CameraGeometry", "EventSlice",
    "EventStream", "EvflowError", "EventParseError", "GeometryError",
    "DimensionMismatchError", "EmptyNeighborhoodError", "TrainConfig", "TrainingDivergedError", "train_head",
]
