"""B200 (sm_100a) hot path of Newson et al., "Video inpainting of complex scenes" (arXiv 1503.05528).

libvinp.so (include/vinp.h) holds every kernel; `vinp` is its ctypes binding and `inpaint` the
Alg. 4 driver.  Exports are resolved lazily so that `paper_1503_05528_b200.build` can run before
the library exists; any use of the binding loads libvinp.so and raises if it is missing (there
is no CPU fallback).
"""
import importlib

_EXPORTS = {"vinp": (".vinp", None), "Config": (".driver", "Config"),
            "Exchange": (".driver", "Exchange"), "Inpainter": (".driver", "Inpainter"),
            "inpaint": (".driver", "inpaint")}


def __getattr__(name):
    if name in _EXPORTS:
        mod, attr = _EXPORTS[name]
        m = importlib.import_module(mod, __name__)
        return m if attr is None else getattr(m, attr)
    raise AttributeError(name)


__all__ = list(_EXPORTS)
