"""B200 hot path of arXiv 1509.04863 (fast template matching, Algorithm 1).

Thin Python binding over the C ABI in ``include/tm.h`` (``libtm.so``, built
in-tree for sm_100a).  This module only marshals arguments: every step of the
path runs in the library's CUDA kernels.  PyTorch supplies device memory and
streams.  There is no CPU fallback: importing works without a GPU (so the
library's exports can be checked), but every compute call needs the CUDA
extension and a CUDA device and raises otherwise.
"""
from __future__ import annotations

import ctypes
import os

from ._binding import (TM_BINARY, TM_CORR_NTT, TM_CORR_TC, TM_F32, TM_I8, Plan, TMError, lib, lib_path,  # noqa: F401
                       EXPORTED_SYMBOLS, RUN_PATHS, MultiPlan, crt_multi, launch_count, profile_events, probe_read_bw)
from .pipeline import Pipeline  # noqa: F401
from .single import SingleSignal  # noqa: F401

__all__ = ["Plan", "MultiPlan", "crt_multi", "TMError", "TM_I8", "TM_F32", "TM_BINARY", "TM_CORR_NTT", "TM_CORR_TC", "lib", "lib_path", "EXPORTED_SYMBOLS",
           "launch_count", "profile_events", "probe_read_bw", "SingleSignal", "Pipeline"]
