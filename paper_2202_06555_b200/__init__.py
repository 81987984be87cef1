"""B200-native evaluation of adaptive sparse-grid / cut-HDMR interpolants
(the hot path of arXiv 2202.06555, DDSG).  See DESIGN.md."""
from .ddsg import (  # noqa: F401
    EXACT,
    FAST,
    MODIFIED_LINEAR,
    ZERO_BOUNDARY,
    BuildError,
    DdsgError,
    DomainError,
    InvalidArgument,
    SparseGridFunction,
    VectorizedDdsg,
    last_eval_stats,
    uniform_points,
)
