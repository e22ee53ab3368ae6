"""B200-native GOFMM evaluation phase (u = K~ W) behind a C-ABI (include/gofmm_b200.h).

Drop-in for gfmm::evaluate (reference: proj/include/gfmm/evaluate.hpp:287-317). The compute path
is the sm_100a extension _lib/libgofmm_b200.so; this package only marshals the compressed tree.
"""
from ._lib import (BLOCKS_MATERIALIZE, BLOCKS_MATRIX_FREE, GOFMM_ERR_CUDA, GOFMM_ERR_INVALID,
                   GOFMM_ERR_IO, GOFMM_ERR_NUMERIC, KERNEL_EXPONENTIAL, KERNEL_GAUSSIAN, KERNEL_LAPLACE,
                   KERNEL_POLYNOMIAL, GofmmError, InvalidArgument, build)
from .gofmm import CompressedTree, Evaluator, Potentials
from .ann import ann_leaf_merge
from .skeleton import Skeleton, skeletonize_batch
from .compress import CompressResult, compress

__all__ = [
    "BLOCKS_MATERIALIZE", "BLOCKS_MATRIX_FREE", "GOFMM_ERR_CUDA", "GOFMM_ERR_INVALID", "GOFMM_ERR_IO",
    "GOFMM_ERR_NUMERIC", "KERNEL_EXPONENTIAL", "KERNEL_GAUSSIAN", "KERNEL_LAPLACE", "KERNEL_POLYNOMIAL",
    "GofmmError", "InvalidArgument", "build", "CompressedTree", "Evaluator", "Potentials", "Skeleton",
    "skeletonize_batch", "ann_leaf_merge", "compress", "CompressResult",
]
