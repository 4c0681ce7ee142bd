"""B200-native dSMC (de-Sequentialized Monte Carlo, arXiv 2202.02264).

The product is the CUDA/C++ engine behind the C ABI in include/dsmc_b200.h
(paper_2202_02264_b200/libdsmc_b200.so). This package is its Python binding
plus host-side model builders; `dsmc` fails loudly when the library is absent.
"""
from . import abi  # noqa: F401  (plain ctypes structs, no library load)

__all__ = ["abi", "dsmc", "models"]
