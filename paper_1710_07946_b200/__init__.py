"""B200-native (sm_100a) superfast CUR low-rank approximation — the data-parallel hot path of
arXiv 1710.07946 (Alg 10.2 with C-A iterations, canonical nucleus, a-posteriori check).

The product is the C-ABI library ``liblra.so`` (include/lra.h) built from ``csrc/``; this
package is its thin ctypes binding (``lra``) plus the end-to-end convenience pipeline
(``pipeline``).  Importing it loads the library and fails loudly if it is missing — there
is no CPU fallback anywhere in the product path.
"""
from . import lra  # noqa: F401
from .lra import (Dense, Factored, Handle, LraError, Multiplier, lra_batch, lra_cross_approx,  # noqa: F401
                  lra_cur_residual, lra_handle_create, lra_preprocess, nccl_unique_id)

lra.lib()   # load now: missing/stale builds surface at import time
