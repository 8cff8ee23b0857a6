"""B200-native SC-4DVAR Gauss-Newton Hessian-product engine (arXiv 2401.15758 hot path).

The compute path is ``_build/libsdv_cuda.so`` (hand-written sm_100a CUDA,
C-ABI in ``include/sdv.h``); this package is its Python host mirror.
"""
from .api import (LANCZOS, MODEL_BURGERS, MODEL_BURGERS_DIRICHLET, MODEL_BVE, NYSTROM, PRIOR_FOURIER,
                  PRIOR_LAPLACIAN, RANDSVD, SINGLEVIEW, DeviceBuffer, PinnedBuffer, Problem, Trajectory,
                  gaussian_matrix, gaussian_vector, init, launch_count, mix_seed, path_counts, path_delta)
from ._lib import LIB_PATH, SdvCudaError, SdvError

__all__ = ["Problem", "Trajectory", "DeviceBuffer", "PinnedBuffer", "init", "launch_count", "path_counts", "path_delta", "mix_seed",
           "gaussian_matrix", "gaussian_vector", "MODEL_BURGERS", "MODEL_BVE", "MODEL_BURGERS_DIRICHLET",
           "PRIOR_FOURIER", "PRIOR_LAPLACIAN", "RANDSVD", "NYSTROM", "SINGLEVIEW", "LANCZOS", "SdvError",
           "SdvCudaError", "LIB_PATH"]
