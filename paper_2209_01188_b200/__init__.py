"""B200-native block-span server hot path of Petals (arXiv 2209.01188).

Drop-in for the reference's (swarmlm) server compute: int8 block executor,
paged KV sessions, wire codec and span-to-span hop, as hand-written sm_100a
CUDA behind the C-ABI in include/petals_b200.h.
"""

from .errors import (  # noqa: F401
    ERR_BAD_REQUEST,
    ERR_BUSY,
    ERR_CAPACITY,
    ERR_DESYNC,
    ERR_GENERIC,
    ERR_UNKNOWN_SESSION,
    ERR_UNKNOWN_TAPE,
    CapacityError,
    InputError,
    RemoteError,
)
from .model import SHAPES, ModelConfig  # noqa: F401

__version__ = "0.1.0"
