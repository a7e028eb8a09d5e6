"""Producer side of the store: magnitude pruning and layer-wise affine
quantisation, vectorised over a batch of same-architecture records.

These produce the quantised + pruned records the decode path consumes
(BASELINE config 2).  Semantics follow the reference's compressor.py
exactly, so records written here are byte-identical to the reference writer's
(tests/test_archive_writer.py):
  * prune_l1  — global stable argsort of |w| (f64) over all weight entries,
                k = floor(r·n + 0.5), mask AND, w *= mask (compressor.py:109-152)
  * quantize  — hidden layers only; scale = (max-min)/(2^b-1) over kept
                weights, zp = round(-min/scale), codes = clip(round(w/scale)+zp),
                w = f32(scale·(codes-zp))·mask; degenerate -> constant
                (compressor.py:155-204)
  * quantize_codes — codes recomputed from the snapped weights
                (compressor.py:207-218), which is what the archive stores.
Single-model wrappers keep the reference's signatures.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import FormatError, InvalidInputError, NumericError, StructuralError
from .net import Architecture, InrModel, LayerWeights

_MODE_BITS = {"affine8": 8, "affine16": 16}


@dataclass(frozen=True)
class LayerQuant:
    """value = scale · (code − zero_point) (compressor.py:68-79)."""

    bits: int
    scale: float
    zero_point: int
    constant: bool = False


@dataclass(frozen=True)
class QuantInfo:
    mode: str
    layers: dict = field(default_factory=dict)

    @property
    def quantized_layers(self) -> set:
        return set(self.layers)


@dataclass
class LayerQuantBatch:
    """Per-record quantisation parameters of one hidden layer."""

    bits: int
    scale: np.ndarray      # f64 [N]
    zero_point: np.ndarray  # i64 [N]
    constant: np.ndarray   # bool [N]


@dataclass
class ModelBatch:
    """N records of one architecture, stored layer-major:
    w[l] [N, out, in] (f32 or f16), b[l] [N, out] f32, mask[l] [N, out, in]."""

    arch: Architecture
    w: list
    b: list
    mask: list
    source_h: int = 0
    source_w: int = 0
    quant_mode: str = "none"
    quant: dict = field(default_factory=dict)  # layer -> LayerQuantBatch

    @property
    def n(self) -> int:
        return self.w[0].shape[0]

    @staticmethod
    def from_models(models) -> "ModelBatch":
        """Stack same-architecture models (reference InrModel objects work)."""
        m0 = models[0]
        arch = Architecture(m0.arch.dims, m0.arch.omega)
        nl = len(arch.dims) - 1
        w = [np.stack([m.layers[l].w for m in models]) for l in range(nl)]
        b = [np.stack([m.layers[l].b for m in models]).astype(np.float32) for l in range(nl)]
        mask = [np.stack([m.mask[l] for m in models]).astype(bool) for l in range(nl)]
        mb = ModelBatch(arch, w, b, mask, int(m0.source_h), int(m0.source_w))
        if m0.quant is not None:
            mb.quant_mode = m0.quant.mode
            for l in m0.quant.layers:
                lqs = [m.quant.layers[l] for m in models]
                mb.quant[l] = LayerQuantBatch(
                    lqs[0].bits,
                    np.array([q.scale for q in lqs], np.float64),
                    np.array([q.zero_point for q in lqs], np.int64),
                    np.array([q.constant for q in lqs], bool))
        return mb

    def model(self, i: int) -> InrModel:
        layers = [LayerWeights(self.w[l][i].copy(), self.b[l][i].copy()) for l in range(len(self.w))]
        masks = [self.mask[l][i].copy() for l in range(len(self.w))]
        quant = None
        if self.quant_mode != "none":
            quant = QuantInfo(self.quant_mode, {
                l: LayerQuant(q.bits, float(q.scale[i]), int(q.zero_point[i]), bool(q.constant[i]))
                for l, q in self.quant.items()})
        return InrModel(self.arch, layers, masks, self.source_h, self.source_w, quant)


def hidden_layer_indices(n_layers: int) -> range:
    """Everything but the first and last layer (compressor.py:155-157)."""
    return range(1, n_layers - 1)


def prune_l1_batch(mb: ModelBatch, ratios, scope: str = "global") -> ModelBatch:
    """L1 prune of every record to its own total zero ratio: ``scope``
    "global" ranks |w| over all matrices jointly, "per_layer" within each
    matrix (compressor.py:108-152)."""
    ratios = np.broadcast_to(np.asarray(ratios, np.float64), (mb.n,))
    if np.any(~((ratios >= 0.0) & (ratios < 1.0))):
        raise InvalidInputError("total_ratio must be in [0, 1)")
    if scope not in ("global", "per_layer"):
        raise InvalidInputError(f"unknown scope {scope!r}")

    def doomed_of(ws):
        mags = np.concatenate([np.abs(w.reshape(mb.n, -1)).astype(np.float64) for w in ws], axis=1)
        total = mags.shape[1]
        order = np.argsort(mags, axis=1, kind="stable")
        rank = np.empty_like(order)
        np.put_along_axis(rank, order, np.arange(total)[None, :].repeat(mb.n, 0), axis=1)
        k = np.floor(ratios * total + 0.5).astype(np.int64)
        return rank < k[:, None]

    sizes = [w.shape[1] * w.shape[2] for w in mb.w]
    if scope == "global":
        doomed = doomed_of(mb.w)
    else:
        doomed = np.concatenate([doomed_of([w]) for w in mb.w], axis=1)
    out_w, out_m = [], []
    off = 0
    for w, m, sz in zip(mb.w, mb.mask, sizes):
        keep = ~doomed[:, off:off + sz].reshape(m.shape) & m
        off += sz
        if not keep.reshape(mb.n, -1).any(axis=1).all():
            bad = float(ratios[int(np.argmin(keep.reshape(mb.n, -1).any(axis=1)))])
            raise StructuralError(f"ratio {bad} would zero an entire layer" +
                                  (f" ({m.shape[1]}x{m.shape[2]})" if scope == "global" else ""))
        out_m.append(keep)
        out_w.append(np.multiply(w, keep))  # w * False -> -0.0 for negative w, as the reference
    return ModelBatch(mb.arch, out_w, [b.copy() for b in mb.b], out_m, mb.source_h, mb.source_w,
                      mb.quant_mode, dict(mb.quant))


def quantize_batch(mb: ModelBatch, mode: str) -> ModelBatch:
    """Layer-wise affine quantisation of the hidden layers of every record."""
    if mode not in _MODE_BITS:
        raise InvalidInputError(f"mode must be one of {sorted(_MODE_BITS)}, got {mode!r}")
    if mb.quant_mode != "none":
        raise FormatError(f"model already quantized ({mb.quant_mode})")
    for i, (w, b) in enumerate(zip(mb.w, mb.b)):
        if not (np.isfinite(w).all() and np.isfinite(b).all()):
            raise NumericError(f"layer {i} contains non-finite weights")
    bits = _MODE_BITS[mode]
    qmax = (1 << bits) - 1
    out_w = [w.copy() for w in mb.w]
    quant = {}
    n = mb.n
    for l in hidden_layer_indices(len(mb.w)):
        w, m = mb.w[l], mb.mask[l]
        w64 = w.reshape(n, -1).astype(np.float64)
        mflat = m.reshape(n, -1)
        any_kept = mflat.any(axis=1)
        mn = np.where(mflat, w64, np.inf).min(axis=1)
        mx = np.where(mflat, w64, -np.inf).max(axis=1)
        const = ~any_kept | (mx == mn)
        with np.errstate(divide="ignore", invalid="ignore"):
            scale = np.where(const, 1.0, (mx - mn) / qmax)
            zpf = np.where(const, 0.0, np.round(-mn / scale))
        const |= ~((zpf >= -(2.0 ** 31)) & (zpf < 2.0 ** 31))
        scale = np.where(const, 1.0, scale)
        zp = np.where(const, 0, zpf).astype(np.int64)
        with np.errstate(divide="ignore", invalid="ignore"):
            codes = np.clip(np.round(w64 / scale[:, None]) + zp[:, None], 0, qmax)
            snapped = (scale[:, None] * (codes - zp[:, None])).astype(w.dtype)
        snapped = np.multiply(snapped, mflat)
        out_w[l] = np.where(const[:, None], w.reshape(n, -1), snapped).reshape(w.shape)
        quant[l] = LayerQuantBatch(bits, scale.astype(np.float64), zp, const)
    return ModelBatch(mb.arch, out_w, [b.copy() for b in mb.b], [m.copy() for m in mb.mask],
                      mb.source_h, mb.source_w, mode, quant)


def quantize_codes_batch(mb: ModelBatch, layer: int) -> np.ndarray:
    """[N, out*in] unsigned codes recomputed from the snapped weights
    (compressor.py:207-218); rows of constant layers are meaningless."""
    q = mb.quant[layer]
    qmax = (1 << q.bits) - 1
    w64 = mb.w[layer].reshape(mb.n, -1).astype(np.float64)
    codes = np.clip(np.round(w64 / q.scale[:, None]) + q.zero_point[:, None], 0, qmax)
    return codes.astype(np.uint8 if q.bits == 8 else np.uint16)


# ---- single-model API with the reference's signatures -----------------------

def prune_l1(model, total_ratio: float, scope: str = "global") -> InrModel:
    if not (0.0 <= total_ratio < 1.0):
        raise InvalidInputError(f"total_ratio must be in [0, 1), got {total_ratio}")
    return prune_l1_batch(ModelBatch.from_models([model]), total_ratio, scope).model(0)


def quantize(model, mode: str) -> InrModel:
    return quantize_batch(ModelBatch.from_models([model]), mode).model(0)


def to_half(model):
    """Cast all weight matrices to float16, biases stay float32 (compressor.py:236-246)."""
    if getattr(model, "quant", None) is not None:
        raise FormatError("cast before quantizing, not after")
    out = model.copy()
    for lw in out.layers:
        lw.w = lw.w.astype(np.float16)
    return out


def check_quant(model) -> None:
    """The metadata check of dequantize (compressor.py:229-232), without the copy."""
    if model.quant is None:
        return
    hidden = set(hidden_layer_indices(len(model.layers)))
    extra = set(model.quant.layers) - hidden
    if extra:
        raise FormatError(f"quantized_layers {sorted(extra)} are not hidden layers")


def dequantize(model):
    """Validate quantisation metadata and drop it (compressor.py:221-235)."""
    if model.quant is None:
        return model
    check_quant(model)
    out = model.copy()
    out.quant = None
    return out


@dataclass(frozen=True)
class PruneSchedule:
    """Piecewise-linear PSNR -> total prune ratio map with saturation
    (compressor.py:20-32)."""

    name: str
    below: float
    pieces: tuple
    above: float


SCHEDULES = {  # compressor.py:36-40
    "cifar": PruneSchedule("cifar", below=0.0, pieces=((30.0, 35.0, 0.05, -1.5),), above=0.25),
    "large": PruneSchedule("large", below=0.2, pieces=((35.0, 40.0, 0.04, -1.2),), above=0.4),
}


def get_schedule(name: str) -> PruneSchedule:
    try:
        return SCHEDULES[name]
    except KeyError:
        raise InvalidInputError(f"unknown schedule {name!r}; have {sorted(SCHEDULES)}") from None


def dynamic_ratio(schedule: PruneSchedule, psnr: float) -> float:
    """compressor.py:50-65."""
    if math.isnan(psnr):
        raise InvalidInputError("psnr is NaN")
    if psnr == math.inf:
        return schedule.above
    for lo, hi, slope, intercept in schedule.pieces:
        if psnr < lo:
            break
        if psnr <= hi:
            return slope * psnr + intercept
    return schedule.below if psnr < schedule.pieces[0][0] else schedule.above


def dynamic_ratio_cifar(psnr: float) -> float:
    """The reference's 'cifar' PSNR->ratio schedule (compressor.py:37-65),
    used only to draw realistic per-record prune ratios for synthetic stores."""
    if math.isnan(psnr):
        raise InvalidInputError("psnr is NaN")
    if psnr < 30.0:
        return 0.0
    if psnr <= 35.0:
        return 0.05 * psnr - 1.5
    return 0.25
