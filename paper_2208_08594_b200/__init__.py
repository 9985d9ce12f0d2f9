"""B200-native MSP-GMRES SOLVE phase (arXiv 2208.08594) — thin Python binding over the
C-ABI library libmsp.so (include/msp.h).  Argument marshalling only: every step of the
solve path runs in the library's sm_100a kernels.  There is no CPU fallback: importing
this package fails loudly when the native library is missing.
"""
from ._binding import (MspError, MspSolver, DistSolver, HostSetup, Config, lib_path, STATUS,  # noqa: F401
                       loopback_solve, nccl_unique_id)

__all__ = ["MspSolver", "DistSolver", "HostSetup", "MspError", "Config", "lib_path", "STATUS",
           "loopback_solve", "nccl_unique_id"]
