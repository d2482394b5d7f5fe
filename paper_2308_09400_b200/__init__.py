"""B200-native (sm_100a) GIPC barrier hot path behind the reference ``tetipc`` entry points.

Importing the package is cheap; the CUDA library (``libb200ipc.so``) is loaded on first use
and must have been built (``python -m paper_2308_09400_b200._build``).  There is no CPU path.
"""

from .barrier import BarrierParams, LocalQuadratic  # noqa: F401
from .proximity import ContactStencil, DistanceResult, StencilKind, StencilTable  # noqa: F401

__version__ = "0.1.0"
