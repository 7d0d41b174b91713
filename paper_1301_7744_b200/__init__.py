"""B200-native BCSS change of basis (arXiv 1301.7744): the ``sttsm_bcss`` hot
path of the reference package ``blocksym`` as hand-written sm_100a FP64
tensor-core CUDA behind the reference's own entry point and tensor object.

Public surface (reference names, /root/reference/pkg/src/blocksym/__init__.py):
``sttsm_bcss``, ``BcssTensor``, ``PartialSymTensor``, ``OpCounter``,
``hypertriangle_iter``, ``simplex_count``, ``canonicalize``, ``DenseTensor``,
``compress`` / ``decompress`` (and the ``_partial`` forms), ``save_bcss`` /
``load_bcss``, ``temp_to_dense``, the error types, plus the device-level
``SttsmPlan`` / ``sttsm_bcss_device``.
"""

from .counters import OpCounter
from .costs import bcss_flops, bcss_memops
from .errors import (
    BlockDivisibilityError,
    ModeError,
    NativeError,
    ParameterError,
    RangeError,
    ShapeError,
    SymmetryError,
)
from .indexing import canonicalize, hypertriangle_iter, hypertriangle_rank, hypertriangle_unrank, simplex_count
from .dense_tensor import DenseTensor, symmetry_violation
from .io import load_bcss, save_bcss
from .storage import (
    BcssTensor,
    PartialSymTensor,
    compress,
    compress_partial,
    decompress,
    decompress_partial,
    packed_payload,
)
from .sttsm import (
    DenseBlockTable,
    SttsmPlan,
    clear_plan_cache,
    probe_fp64_peak,
    sttsm_bcss,
    sttsm_bcss_device,
    temp_to_dense,
)

__version__ = "0.1.0"
