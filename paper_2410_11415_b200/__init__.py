"""paper_2410_11415_b200: B200-native evaluation path of KLay layered circuits.

Drop-in for the reference's evaluation engine (``laycirc.engine``): the same
public names, evaluated by hand-written sm_100a kernels in ``libklay.so``.
Circuit construction / layerization stay with the reference (out of scope);
any reference ``TensorizedCircuit`` can be passed in unchanged, or loaded
with ``read_klay`` / ``load_npz`` from this package.
"""

from .engine import (
    BOOLEAN,
    MAX_PRODUCT,
    REAL,
    SEMIRINGS,
    DevicePlan,
    EvalError,
    EvalTrace,
    Semiring,
    WeightAssignment,
    backward,
    clear_cache,
    device_plan,
    evaluate_semiring,
    forward_log,
    forward_real,
    gradient,
    weights_from_json,
    weights_from_map,
    weights_from_probabilities,
)
from .tensorized import (
    KlayFormatError,
    Literal,
    TensorizedCircuit,
    TensorLayer,
    load_npz,
    read_klay,
    save_npz,
    stats,
    write_klay,
)

__version__ = "0.1.0"


def __getattr__(name):  # torch surface, imported lazily (torch is heavy)
    if name in ("CircuitModule", "KlayFunction"):
        from . import torch_module
        return getattr(torch_module, name)
    raise AttributeError(name)

__all__ = [
    "BOOLEAN", "CircuitModule", "KlayFunction", "MAX_PRODUCT", "REAL", "SEMIRINGS", "DevicePlan",
    "EvalError", "EvalTrace",
    "KlayFormatError", "Literal", "Semiring", "TensorLayer", "TensorizedCircuit",
    "WeightAssignment", "backward", "clear_cache", "device_plan", "evaluate_semiring", "forward_log",
    "forward_real", "gradient", "load_npz", "read_klay", "save_npz", "stats",
    "weights_from_json", "weights_from_map", "weights_from_probabilities", "write_klay",
]
