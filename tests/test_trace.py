"""NVTX stage ranges (paper_2306_16699_b200/trace.py): off by default, nest
and unwind on exceptions when on.  CPU-only: torch's NVTX bindings load
without a GPU."""

import pytest
import torch

from paper_2306_16699_b200 import trace


def test_off_by_default_is_a_no_op(monkeypatch):
    calls = []
    monkeypatch.setattr(torch.cuda.nvtx, "range_push", lambda n: calls.append(("push", n)))
    monkeypatch.setattr(torch.cuda.nvtx, "range_pop", lambda: calls.append(("pop",)))
    prev = trace.enabled()
    trace.enable(False)
    try:
        with trace.stage("forward"):
            pass
    finally:
        trace.enable(prev)
    assert calls == []


def test_ranges_nest_and_pop_on_error(monkeypatch):
    calls = []
    monkeypatch.setattr(torch.cuda.nvtx, "range_push", lambda n: calls.append(("push", n)))
    monkeypatch.setattr(torch.cuda.nvtx, "range_pop", lambda: calls.append(("pop",)))
    prev = trace.enabled()
    trace.enable(True)
    try:
        with trace.stage("load"):
            with pytest.raises(ValueError):
                with trace.stage("dequantize"):
                    raise ValueError("x")
    finally:
        trace.enable(prev)
    assert calls == [("push", "rinr.load"), ("push", "rinr.dequantize"), ("pop",), ("pop",)]


def test_real_nvtx_calls_do_not_need_a_gpu():
    prev = trace.enabled()
    trace.enable(True)
    try:
        with trace.stage("forward"):
            pass
    finally:
        trace.enable(prev)
