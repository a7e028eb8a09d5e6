"""NVTX ranges over the decode pipeline's stages (SURVEY.md §5 tracing).

The reference times its pipeline with host stage timers — load, dequantize,
forward, clamp_convert (``pkg/src/rinr/bench.py:39-70``).  Here the same
stages are NVTX ranges, so an ncu capture can be filtered to one stage
(``ncu --nvtx --nvtx-include "rinr.forward/"``; ncu reads "/" as
nesting, so names use "." as the separator) and the stage names line up
with ``harness.bench``'s ``stage_seconds`` keys.

Ranges are off by default: a push/pop pair costs ~1 µs of host time on the
small-batch drop-in path.  ``RINR_NVTX=1`` in the environment (read once at
import) or ``enable(True)`` turns them on.  Names are prefixed ``rinr.``.
"""

from __future__ import annotations

import contextlib
import os

import torch

_on = os.environ.get("RINR_NVTX", "0") not in ("", "0")


def enable(flag: bool = True) -> None:
    global _on
    _on = bool(flag)


def enabled() -> bool:
    return _on


@contextlib.contextmanager
def stage(name: str):
    """``with stage("forward"): ...`` -> NVTX range ``rinr.forward``."""
    if not _on:
        yield
        return
    torch.cuda.nvtx.range_push("rinr." + name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()
