"""B200-native (sm_100a) OmniSparse sparse-attention hot path.

Reference-facing operator API (names of ``slimattn``): :mod:`.prefill`,
:mod:`.decode`; device composite: :mod:`.pipeline`; raw ops over the C ABI
(``include/omnisparse.h``): :mod:`.ops`. The CUDA library is loaded lazily on
first use; there is no CPU fallback.
"""

from .errors import (  # noqa: F401
    DegenerateContextError,
    DegenerateRowError,
    IntegrityError,
    LayoutError,
    ParameterError,
    ShapeError,
    SlimAttnError,
)

__version__ = "0.1.0"
