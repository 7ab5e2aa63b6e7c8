"""B200-native hot path of Allan-Poe (arxiv 2511.00855): the hybrid distance
kernel, GPU graph construction (NN-Descent + RNG-IP pruning + keyword
recycling) and batched beam search, behind the reference's fusegraph API.

Compute lives in libfgb200.so (CUDA, sm_100a) behind the C-ABI of
include/fg_b200.h; this package is the thin Python mirror of the API."""
from ._lib import Error, device_count, lib  # noqa: F401
from . import _abi as abi  # noqa: F401
