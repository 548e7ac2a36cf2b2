"""B200-native (sm_100a) HSDE-ADMM hot path for SOS-derived SDPs (arXiv 1708.04174).

The product path is the CUDA library `libsosadmm.so` (C ABI: include/sosadmm.h) and the thin
ctypes binding `SosAdmm`.  It never imports `oracle/`."""
from .sosadmm import EXPORTS, LIB_PATH, STATUS, SosAdmm, iterate_batch, load_library  # noqa: F401
