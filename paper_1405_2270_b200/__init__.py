"""latsum on B200: the assembled canonical-tensor lattice summation of
arXiv 1405.2270 (generator -> assembled O(N L R) sum -> FP64 rank-R expansion
onto the N^3 grid -> functionals) as hand-written sm_100a CUDA behind a C ABI
(include/latsum_cuda.h) and a drop-in of the reference's C++ API
(include/latsum/*.hpp). This package is the Python mirror of that API.
"""
from ._abi import CudaError, ResourceGuardError, ValidationError, load as load_library  # noqa: F401
from .latsum import *  # noqa: F401,F403
from .latsum import (CanonicalTensor3, Charge, DevicePipeline, GaussianBasisSpec, GridSpec,  # noqa: F401
                     LatticeSpec, QuadratureRule, SumResult)
