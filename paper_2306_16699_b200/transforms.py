"""GPU model transforms of the encode pipeline:
``prune_l1``, ``quantize`` (+ codes) and ``psnr`` over a device-resident batch
of same-architecture models, through the C ABI in
``include/rinr_b200_transforms.h`` (kernels: ``csrc/transforms.cu``).

Each function mirrors the reference function of the same name and gives
bit-identical weights, masks, scales, zero points and codes:

  * ``compressor.prune_l1``:       ``compressor.py:108-152``
  * ``compressor.quantize``:       ``compressor.py:160-202``
  * ``compressor.quantize_codes``: ``compressor.py:205-218``
  * ``metrics.psnr``:              ``metrics.py:23-41`` (f64; summation order differs)

Errors follow the reference's exception types.  A failing model raises
``BatchItemError(i, cause)`` naming the first failing index, as
``decode_batch`` does.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import errors as E
from .compressor import LayerQuantBatch, ModelBatch, hidden_layer_indices
from .errors import BatchItemError, FormatError, InvalidInputError, NumericError, StructuralError
from .net import Architecture

_MODE_BITS = {"affine8": 8, "affine16": 16}


@dataclass
class DeviceModels:
    """N models of one architecture on the GPU, in the transform layout:
    ``w`` [N, P] f32 (matrices concatenated, each row-major (out, in)),
    ``mask`` [N, P] u8, ``b`` [N, sum(out)] f32."""

    arch: Architecture
    w: torch.Tensor
    mask: torch.Tensor
    b: torch.Tensor
    source_h: int = 0
    source_w: int = 0

    @property
    def n(self) -> int:
        return self.w.shape[0]

    @property
    def sizes(self) -> list:
        d = self.arch.dims
        return [d[l] * d[l + 1] for l in range(len(d) - 1)]

    @staticmethod
    def from_batch(mb: ModelBatch, device="cuda") -> "DeviceModels":
        if any(w.dtype != np.float32 for w in mb.w):
            raise InvalidInputError("GPU transforms take float32 weights (cast after quantizing, not before)")
        n = mb.n
        w = np.concatenate([w.reshape(n, -1) for w in mb.w], axis=1)
        m = np.concatenate([m.reshape(n, -1) for m in mb.mask], axis=1).astype(np.uint8)
        b = np.concatenate([b.reshape(n, -1) for b in mb.b], axis=1).astype(np.float32)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
        return DeviceModels(mb.arch, t(w), t(m), t(b), mb.source_h, mb.source_w)

    def to_batch(self) -> ModelBatch:
        d = self.arch.dims
        n = self.n
        w = self.w.cpu().numpy()
        m = self.mask.cpu().numpy().astype(bool)
        b = self.b.cpu().numpy()
        ws, ms, bs, off, boff = [], [], [], 0, 0
        for l in range(len(d) - 1):
            sz = d[l] * d[l + 1]
            ws.append(w[:, off:off + sz].reshape(n, d[l + 1], d[l]).copy())
            ms.append(m[:, off:off + sz].reshape(n, d[l + 1], d[l]).copy())
            bs.append(b[:, boff:boff + d[l + 1]].copy())
            off += sz
            boff += d[l + 1]
        return ModelBatch(self.arch, ws, bs, ms, self.source_h, self.source_w)


def _dims(arch: Architecture):
    return (C.c_int32 * len(arch.dims))(*arch.dims), len(arch.dims) - 1


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _raise_items(status: torch.Tensor, what: str) -> None:
    s = status.cpu().numpy()
    bad = np.nonzero(s)[0]
    if bad.size:
        i = int(bad[0])
        code = int(s[i])
        cause = {E.ERR_STRUCTURAL: StructuralError, E.ERR_NUMERIC: NumericError,
                 E.ERR_INVALID_INPUT: InvalidInputError}.get(code, FormatError)(f"{what} failed (status {code})")
        raise BatchItemError(i, cause)


def prune_l1(dm: DeviceModels, total_ratio, scope: str = "global", check: bool = True) -> torch.Tensor:
    """In-place magnitude prune of every model to its own total zero ratio
    (``total_ratio``: scalar or [N]).  Returns the per-model status tensor;
    with ``check`` raises ``BatchItemError`` for the first failing model
    (whose weights and mask are left unchanged)."""
    if scope not in ("global", "per_layer"):
        raise InvalidInputError(f"unknown scope {scope!r}")
    r = torch.as_tensor(total_ratio, dtype=torch.float64).expand(dm.n).contiguous().to(dm.w.device)
    status = torch.zeros(dm.n, dtype=torch.int32, device=dm.w.device)
    dims, nl = _dims(dm.arch)
    with torch.cuda.device(dm.w.device):  # launch on the tensors' device
        N.check(N.lib().rinr_prune_l1(dims, nl, dm.n, dm.w.data_ptr(), dm.mask.data_ptr(), r.data_ptr(),
                                      0 if scope == "global" else 1, status.data_ptr(), _stream(dm.w.device)))
    if check:
        _raise_items(status, "prune_l1")
    return status


@dataclass
class DeviceQuant:
    """Per-(model, hidden layer) quantisation results; ``codes`` [N, P] u16
    holds the codes of every entry of the quantised (non-constant) matrices."""

    mode: str
    bits: int
    scale: torch.Tensor  # f64 [N, nl-2]
    zero_point: torch.Tensor  # i32 [N, nl-2]
    constant: torch.Tensor  # bool [N, nl-2]
    codes: torch.Tensor
    status: torch.Tensor

    def layer_quant(self) -> dict:
        s, z, c = self.scale.cpu().numpy(), self.zero_point.cpu().numpy(), self.constant.cpu().numpy()
        return {h + 1: LayerQuantBatch(self.bits, s[:, h].copy(), z[:, h].astype(np.int64), c[:, h].astype(bool))
                for h in range(s.shape[1])}


def quantize(dm: DeviceModels, mode: str, check: bool = True) -> DeviceQuant:
    """In-place layer-wise affine quantisation of the hidden matrices."""
    if mode not in _MODE_BITS:
        raise InvalidInputError(f"mode must be one of {sorted(_MODE_BITS)}, got {mode!r}")
    bits = _MODE_BITS[mode]
    dev = dm.w.device
    nh = max(len(dm.arch.dims) - 3, 0)
    scale = torch.ones((dm.n, nh), dtype=torch.float64, device=dev)
    zp = torch.zeros((dm.n, nh), dtype=torch.int32, device=dev)
    const = torch.zeros((dm.n, nh), dtype=torch.uint8, device=dev)
    codes = torch.zeros_like(dm.w, dtype=torch.int16)  # u16 payload (torch has no uint16 arithmetic)
    status = torch.zeros(dm.n, dtype=torch.int32, device=dev)
    dims, nl = _dims(dm.arch)
    with torch.cuda.device(dm.w.device):  # launch on the tensors' device
        N.check(N.lib().rinr_quantize(dims, nl, dm.n, bits, dm.w.data_ptr(), dm.mask.data_ptr(), dm.b.data_ptr(),
                                      scale.data_ptr(), zp.data_ptr(), const.data_ptr(), codes.data_ptr(),
                                      status.data_ptr(), _stream(dev)))
    if check:
        _raise_items(status, "quantize")
    return DeviceQuant(mode, bits, scale, zp, const.bool(), codes, status)


def quantized_batch(dm: DeviceModels, q: DeviceQuant) -> ModelBatch:
    """Host ModelBatch of the quantised models (what archive.serialize_batch
    writes): weights, masks, biases and the per-layer quant parameters."""
    mb = dm.to_batch()
    mb.quant_mode = q.mode
    mb.quant = q.layer_quant()
    return mb


def psnr(a: torch.Tensor, b: torch.Tensor, quantized: bool = False):
    """Per-image (mse, psnr_db) f64 tensors for [N, ...] f32 batches in [0, 1]."""
    if a.shape != b.shape or a.dim() < 1:
        raise InvalidInputError(f"dimension mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    a = a.to(torch.float32).contiguous()
    b = b.to(device=a.device, dtype=torch.float32).contiguous()
    n = a.shape[0]
    count = a[0].numel() if n else 1
    mse = torch.empty(n, dtype=torch.float64, device=a.device)
    out = torch.empty(n, dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):  # launch on the tensors' device
        N.check(N.lib().rinr_psnr(a.data_ptr(), b.data_ptr(), n, count, int(quantized), mse.data_ptr(), out.data_ptr(),
                                  _stream(a.device)))
    return mse, out


def serialize(dm: DeviceModels, q: DeviceQuant | None = None, id_prefix: str = "img", first_id: int = 0,
              id_width: int = 8) -> torch.Tensor:
    """Archive bytes of the batch as a device uint8 tensor, written on the GPU
    (csrc/writer.cu) and byte-identical to ``archive.serialize_batch`` of the
    same models (the reference writer, archive.py:92-184).  Record k's id is
    ``f"{id_prefix}{first_id + k:0{id_width}d}"``; ``q`` is the result of
    ``quantize`` on these models (None: unquantised f32 records)."""
    dev = dm.w.device
    n = dm.n
    dims, nl = _dims(dm.arch)
    a = N.SerializeArgs()
    a.dims = C.cast(dims, C.POINTER(C.c_int32))
    a.n_layers = nl
    a.n = n
    a.source_h, a.source_w = int(dm.source_h), int(dm.source_w)
    a.omega = float(dm.arch.omega)
    a.quant_bits = q.bits if q is not None else 0
    a.d_w, a.d_mask, a.d_b = dm.w.data_ptr(), dm.mask.data_ptr(), dm.b.data_ptr()
    if q is not None:
        a.d_scale, a.d_zp = q.scale.data_ptr(), q.zero_point.data_ptr()
        const_u8 = q.constant.to(torch.uint8).contiguous()
        a.d_const, a.d_codes = const_u8.data_ptr(), q.codes.data_ptr()
    a.id_prefix = id_prefix.encode("utf-8")
    a.first_id = int(first_id)
    a.id_width = int(id_width)
    rec_len = torch.empty(n, dtype=torch.int64, device=dev)
    forms = torch.empty((n, nl), dtype=torch.uint8, device=dev)
    kept = torch.empty((n, nl), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = _stream(dev)
        N.check(N.lib().rinr_serialize_size(C.byref(a), rec_len.data_ptr(), forms.data_ptr(), kept.data_ptr(), st))
        ends = torch.cumsum(rec_len, 0)
        total = int(ends[-1].item()) if n else 0
        rec_off = ends - rec_len
        out = torch.empty(10 + 12 * n + total, dtype=torch.uint8, device=dev)
        N.check(N.lib().rinr_serialize_write(C.byref(a), rec_off.data_ptr(), rec_len.data_ptr(), forms.data_ptr(),
                                             kept.data_ptr(), out.data_ptr(), st))
    return out


__all__ = ["DeviceModels", "DeviceQuant", "prune_l1", "quantize", "quantized_batch", "psnr", "serialize",
           "hidden_layer_indices"]
