"""B200-native differentiable DF-II / TDF-II IIR filtering (arXiv 2511.14390).

The compute path is the C-ABI library ``libiirgrad.so`` (hand-written sm_100a
CUDA, see ``include/iirgrad.h``); this package is a thin binding over it.
Importing the package does not load the library; the first call does, and it
fails loudly if the library is missing -- there is no CPU fallback.
"""
__all__ = ["lfilter", "allpole_tv", "lfilter_tv", "matrix_recurrence", "iir_forward", "iir_backward"]


def __getattr__(name):
    if name in ("lfilter", "LFilterFunction", "allpole_tv", "AllPoleTVFunction", "lfilter_tv", "TVDFFunction",
                "matrix_recurrence", "LTIMatrixRecurrenceFunction"):
        from . import autograd
        return getattr(autograd, name)
    if name in ("iir_forward", "iir_backward", "Desc", "lib"):
        from . import _binding
        return getattr(_binding, name)
    raise AttributeError(name)
