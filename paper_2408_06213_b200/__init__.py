"""B200-native batched dice rolls and segmented Fisher-Yates shuffles (arXiv 2408.06213).

The hot path of the reference package ``batchrand`` re-built for sm_100a: a device PCG64,
a bulk batched-roll kernel and size-dispatched segmented shuffle kernels behind a C ABI
(include/batchrand_b200.h), with a drop-in Python API in ``.batchrand``.
"""

from .batchrand import *  # noqa: F401,F403
from .batchrand import __all__ as _core_all
from .cost_model import CostParams, build_schedule, cost_per_roll, find_nk  # noqa: F401
from .errors import InsufficientTrials, NoCrossover, UnknownAlgorithm  # noqa: F401
from .multi import roll_batches_sharded, shuffle_many_sharded  # noqa: F401

__all__ = list(_core_all) + ["CostParams", "build_schedule", "cost_per_roll", "find_nk", "InsufficientTrials",
                             "NoCrossover", "UnknownAlgorithm", "roll_batches_sharded", "shuffle_many_sharded"]

__version__ = "0.1.0"
