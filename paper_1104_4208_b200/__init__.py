"""B200-native DG Maxwell hot path of arXiv:1104.4208 (product package).

``libdgm.so`` (CUDA, sm_100a) implements the C ABI of include/dgm.h;
``binding.Context`` is the thin ctypes layer over it.  The package never imports
the test oracle (``oracle/``) and has no CPU fallback.
"""
from .binding import Context, DgmError, load_library  # noqa: F401
