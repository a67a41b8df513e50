"""paper_2003_07065_b200 -- B200-native fast downsampled SST (He & Cao, arXiv 2003.07065).

The product is ``libsst.so`` (C ABI in include/sst.h, hand-written sm_100a CUDA).  This
package is its thin Python binding: ``Plan`` (forward / inverse / debug entry points) and
``dist`` (time sharding over ranks with torch.distributed).  Importing it raises if the
library has not been built; there is no fallback path.
"""

from ._lib import (  # noqa: F401
    SSTError, SST_OK, SST_E_INVALID_ARGUMENT, SST_E_COVERAGE, SST_E_UNSUPPORTED, SST_E_CUDA,
    SST_E_OUT_OF_MEMORY, SST_E_INTERNAL, SST_GAMMA_RELATIVE, SST_SOURCE_TRUNCATE, SST_DETERMINISTIC,
    SST_DISCRETE_CONSTANT, SST_FILTER_BANK, SST_WARN_EQ37, SST_WARN_EQ46, SST_PATH_FUSED,
    SST_PATH_MULTIPASS, SST_PATH_FILTERBANK, SST_IPATH_RESIDUE, SST_IPATH_NARROWBAND, SST_IPATH_MULTIPASS, LIB_PATH,
)
from .plan import Plan, gaussian_window, make_params, validate, layout, gamma_bound  # noqa: F401

__version__ = "0.1.0"
