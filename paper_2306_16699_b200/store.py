"""``Store``: an HBM-resident .rinr dataset and the batched decode over it.

This is the training-loop face of the decode path: the whole
INR dataset is moved to device memory once and every batch is
decoded on the fly by one fused kernel launch.  Python only marshals
arguments; parsing, dequantisation, the MLP and the epilogue are native
(csrc/).  torch supplies device memory and streams.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .errors import BatchItemError, InvalidInputError
from .trace import stage

_DTYPES = {torch.float32: N.OUT_F32, torch.bfloat16: N.OUT_BF16, torch.uint8: N.OUT_U8}
_PREC = {"fp32": N.PREC_FP32, "bf16": N.PREC_BF16, "exact": N.PREC_EXACT}
_SIN = {"mufu": N.SIN_MUFU, "accurate": N.SIN_ACCURATE}
_AUG = {None: N.AUG_NONE, "none": N.AUG_NONE, "offset": N.AUG_OFFSET, "crop": N.AUG_CROP}


class Store:
    """Immutable device-resident store built from .rinr bytes (or a path).

    ``shard_rank/shard_world`` keep records with ``k % world == rank``; ids
    passed to ``decode`` are local indices into the shard (global index of
    local i = i * world + rank)."""

    def __init__(self, source, device=None, shard_rank: int = 0, shard_world: int = 1):
        if isinstance(source, (str, Path)):
            source = Path(source).read_bytes()
        dev = torch.device("cuda") if device is None else torch.device(device)
        if dev.type != "cuda":
            raise InvalidInputError("Store lives in GPU memory; device must be a CUDA device")
        if dev.index is None:  # "cuda" means the current device (e.g. after set_device(local_rank))
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        arr = N.host_view(source)
        h = C.c_void_p()
        with stage("load"):
            N.check(N.lib().rinr_store_create(arr.ctypes.data if arr.size else None, arr.size, dev.index,
                                              shard_rank, shard_world, C.byref(h)))
        self._h = h
        info = N.StoreInfo()
        N.check(N.lib().rinr_store_info(self._h, C.byref(info)))
        self.info = info
        self.dims = tuple(info.dims[: info.n_dims])
        self._status = torch.zeros(1, dtype=torch.int32, device=dev)

    # -- metadata -----------------------------------------------------------
    def __len__(self) -> int:
        return int(self.info.num_records)

    @property
    def handle(self) -> int:
        return self._h.value

    def record_meta(self, k: int) -> dict:
        g = C.c_int64()
        buf = C.create_string_buffer(256)
        n = C.c_size_t()
        sh, sw = C.c_uint32(), C.c_uint32()
        N.check(N.lib().rinr_store_record_meta(self._h, k, C.byref(g), buf, 256, C.byref(n), C.byref(sh),
                                               C.byref(sw)))
        rid = buf.value.decode("utf-8")
        if n.value >= 256:
            buf = C.create_string_buffer(n.value + 1)
            N.check(N.lib().rinr_store_record_meta(self._h, k, None, buf, n.value + 1, None, None, None))
            rid = buf.value.decode("utf-8")
        return {"global_index": g.value, "id": rid, "source_h": sh.value, "source_w": sw.value}

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            h, self._h = self._h, C.c_void_p()  # the handle is freed even if cudaFree reports an error
            N.check(N.lib().rinr_store_destroy(h))

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- kernels ------------------------------------------------------------
    def _ids(self, ids) -> torch.Tensor:
        if not isinstance(ids, torch.Tensor):
            ids = torch.as_tensor(np.asarray(ids, dtype=np.int64))
        return ids.to(device=self.device, dtype=torch.int64).contiguous()

    def _raise_status(self, n: int) -> None:
        bad = int(self._status.item())
        if bad:
            i = n - bad
            raise BatchItemError(i, InvalidInputError(f"record id out of range [0, {len(self)})"))

    def dequantize(self, ids, check: bool = True) -> torch.Tensor:
        """[n, max_param_count] f32: materialised [w0, b0, w1, b1, ...] per id
        (bit-exact with archive.materialize)."""
        ids = self._ids(ids)
        n = ids.numel()
        P = int(self.info.max_param_count)
        out = torch.empty((n, P), dtype=torch.float32, device=self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        with stage("dequantize"):
            N.check(N.lib().rinr_dequantize(self._h, ids.data_ptr(), n, out.data_ptr(), P,
                                            self._status.data_ptr() if check else None, stream))
        if check:
            self._raise_status(n)
        return out

    def decode_params(self, out_h, out_w, dtype=torch.float32, layout="nchw", precision="fp32", sin="mufu",
                      aug_mode=None, mean=None, std=None, overlap_prologue: bool = False,
                      prefetch_next: bool = False) -> N.DecodeParams:
        """``overlap_prologue``: promise that ids/aug were not written by the
        kernel launched just before this decode on the stream, letting the
        record fetch + dequantisation overlap that kernel's tail (PDL).
        ``prefetch_next``: every decode with these params passes ``next_ids``
        (RINR_FLAG_PREFETCH_NEXT)."""
        if out_h is None or out_w is None:
            if not self.info.uniform_source:
                raise InvalidInputError("records differ in source size; pass out_h and out_w")
            out_h = self.info.source_h if out_h is None else out_h
            out_w = self.info.source_w if out_w is None else out_w
        p = N.DecodeParams()
        p.out_h, p.out_w = int(out_h), int(out_w)
        if dtype not in _DTYPES:
            raise InvalidInputError(f"unsupported output dtype {dtype}")
        p.out_dtype = _DTYPES[dtype]
        p.out_layout = {"nchw": N.LAYOUT_NCHW, "nhwc": N.LAYOUT_NHWC}[layout]
        p.precision = _PREC[precision]
        p.sin_mode = _SIN[sin]
        p.aug_mode = _AUG[aug_mode]
        p.mean[:] = list(mean) if mean is not None else [0.0, 0.0, 0.0]
        p.std[:] = list(std) if std is not None else [1.0, 1.0, 1.0]
        p.flags = (N.FLAG_OVERLAP_PROLOGUE if overlap_prologue else 0) | (N.FLAG_PREFETCH_NEXT if prefetch_next else 0)
        return p

    def decode(self, ids, out_h=None, out_w=None, *, out=None, dtype=torch.float32, layout="nchw",
               precision="fp32", sin="mufu", aug=None, aug_mode=None, mean=None, std=None,
               check=True, params=None, next_ids=None) -> torch.Tensor:
        """Decode ``ids`` (local indices) into [n,3,H,W] (nchw) or [n,H,W,3]
        (nhwc).  ``aug``: [n,5] f32 per-image crop/flip parameters for
        ``aug_mode`` 'offset' or 'crop' (see include/rinr_b200.h).
        ``next_ids``: the next batch's n ids (already written on the device);
        their records are prefetched into L2 during this decode.  Zero-copy
        when they directly follow ``ids`` in memory (rows of one tensor)."""
        ids = self._ids(ids)
        n = ids.numel()
        if params is None:
            params = self.decode_params(out_h, out_w, dtype, layout, precision, sin, aug_mode, mean, std,
                                        prefetch_next=next_ids is not None)
        if bool(params.flags & N.FLAG_PREFETCH_NEXT) != (next_ids is not None):
            raise InvalidInputError("next_ids must be passed exactly when the params carry prefetch_next")
        if next_ids is not None:
            nxt = self._ids(next_ids)
            if nxt.numel() != n:
                raise InvalidInputError(f"next_ids must hold {n} ids, got {nxt.numel()}")
            if (n and nxt.data_ptr() == ids.data_ptr() + 8 * n
                    and nxt.untyped_storage().data_ptr() == ids.untyped_storage().data_ptr()):
                ids = ids.as_strided((2 * n,), (1,))
            else:
                ids = torch.cat([ids, nxt])
        H, W = params.out_h, params.out_w
        shape = (n, 3, H, W) if params.out_layout == N.LAYOUT_NCHW else (n, H, W, 3)
        tdtype = {N.OUT_F32: torch.float32, N.OUT_BF16: torch.bfloat16, N.OUT_U8: torch.uint8}[params.out_dtype]
        if out is None:
            out = torch.empty(shape, dtype=tdtype, device=self.device)
        elif out.shape != shape or out.dtype != tdtype or not out.is_contiguous() or out.device != self.device:
            raise InvalidInputError(f"out must be a contiguous {tdtype} tensor of shape {shape} on {self.device}")
        aug_ptr = None
        if params.aug_mode != N.AUG_NONE:
            if aug is None:
                raise InvalidInputError("aug parameters required for this aug_mode")
            aug = aug.to(device=self.device, dtype=torch.float32).contiguous()
            if aug.shape != (n, 5):
                raise InvalidInputError(f"aug must be [n, 5], got {tuple(aug.shape)}")
            aug_ptr = aug.data_ptr()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        with stage("forward"):
            N.check(N.lib().rinr_decode(self._h, ids.data_ptr(), n, C.byref(params), aug_ptr, out.data_ptr(),
                                        self._status.data_ptr() if check else None, stream))
        if check:
            self._raise_status(n)
        return out


# -- augmentation parameter helpers (per-image rows for Store.decode) ---------

def pad_crop_params(n: int, pad: int = 4, generator: torch.Generator | None = None) -> torch.Tensor:
    """CIFAR-style RandomCrop(size, padding=pad) + horizontal flip: rows
    {dx, dy, flip, pad, 0} with dx, dy ~ U{0..2*pad}, flip ~ Bernoulli(0.5).
    Generated on the generator's device (a CUDA generator keeps a training
    loop free of per-step host->device copies)."""
    g = generator
    dev = g.device if g is not None else None
    d = torch.randint(0, 2 * pad + 1, (n, 2), generator=g, device=dev).float()
    flip = torch.randint(0, 2, (n, 1), generator=g, device=dev).float()
    return torch.cat([d, flip, torch.full((n, 1), float(pad), device=dev), torch.zeros(n, 1, device=dev)], 1)


def resized_crop_params(n: int, scale=(0.08, 1.0), ratio=(3 / 4, 4 / 3),
                        generator: torch.Generator | None = None) -> torch.Tensor:
    """RandomResizedCrop + flip as continuous crop boxes in normalised source
    coordinates: rows {x0, y0, sx, sy, flip}.  The INR is sampled directly at
    the crop's output grid, so no resampling happens.  Generated on the
    generator's device."""
    g = generator
    dev = g.device if g is not None else None
    area = torch.empty(n, device=dev).uniform_(scale[0], scale[1], generator=g)
    logr = torch.empty(n, device=dev).uniform_(float(np.log(ratio[0])), float(np.log(ratio[1])), generator=g)
    r = torch.exp(logr)
    sx = torch.sqrt(area * r).clamp(max=1.0)
    sy = torch.sqrt(area / r).clamp(max=1.0)
    x0 = torch.rand(n, generator=g, device=dev) * (1.0 - sx)
    y0 = torch.rand(n, generator=g, device=dev) * (1.0 - sy)
    flip = torch.randint(0, 2, (n,), generator=g, device=dev).float()
    return torch.stack([x0, y0, sx, sy, flip], 1)


IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)
CIFAR_MEAN = (0.4914, 0.4822, 0.4465)
CIFAR_STD = (0.2470, 0.2435, 0.2616)
