"""B200 (sm_100a) hot path of Newson et al., "Video inpainting of complex scenes" (arXiv 1503.05528).

libvinp.so (include/vinp.h) holds every kernel; `vinp` is its ctypes binding and `inpaint`
the Alg. 4 driver.  Importing this package loads libvinp.so and raises if it is missing.
"""
from . import vinp  # noqa: F401  (loads libvinp.so; no fallback)
from .inpaint import Config, Exchange, Inpainter, inpaint  # noqa: F401
