"""paper_2212_09005_b200: B200-native (sm_100a) two-choice filter and counting
quotient filter, a drop-in for the reference package ``filterkit``
(/root/reference/pkg/src/filterkit/__init__.py:14-35).

Same public names: Tcf, TcfParams, BulkTcf, BulkTcfParams, Gqf, GqfParams,
Placement, FilterFullError, CapacityError, ValidationError,
available_backends, __version__.  The single backend is the CUDA library
libfkb200.so (C ABI: include/filterkit_b200.h); there is no CPU fallback.
"""

from .errors import CapacityError, FilterFullError, ValidationError
from .tcf import Placement, Tcf, TcfParams

__version__ = "0.1.0"


def available_backends():
    """The one backend this build has (the reference lists 'c'/'py')."""
    return ["cuda"]


def __getattr__(name):  # lazy: the bulk TCF / GQF modules pull in more kernels
    if name in ("BulkTcf", "BulkTcfParams"):
        from . import tcf_bulk
        return getattr(tcf_bulk, name)
    if name in ("Gqf", "GqfParams"):
        from . import gqf
        return getattr(gqf, name)
    raise AttributeError(name)


__all__ = ["Tcf", "TcfParams", "BulkTcf", "BulkTcfParams", "Gqf", "GqfParams", "Placement",
           "FilterFullError", "CapacityError", "ValidationError", "available_backends",
           "__version__"]
