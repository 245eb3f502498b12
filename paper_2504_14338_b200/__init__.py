"""B200-native dOpInf snapshot pass (arXiv 2504.14338's data-parallel core).

The product is the sm_100a extension libdopinf_b200.so behind the C ABI in
include/dopinf_b200.h; `api` mirrors the reference's stage functions over it.
"""
from . import api  # noqa: F401

__all__ = ["api"]
