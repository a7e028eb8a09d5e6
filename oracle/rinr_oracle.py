"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the Rapid-INR reference's decode path
(``/root/reference/pkg/src/rinr``; citations below are relative to that
directory).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs may import this module, and only as
the checker or the timed CPU baseline.  The CUDA product path never calls it.

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the real
reference package in the build container and records its outputs
(coordinate grids, materialised weights, decoded pixels, archive bytes) in
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` requires this module to
reproduce every one of them bit-for-bit.

What is restated (reference file:line):
  * coordinate grid ........ net.py:138-149
  * forward / trace ........ net.py:183-214
  * decode / decode_batch .. decoder.py:19-61   (clip + HWC reshape, decoder.py:35)
  * u8 conversion .......... image.py:49-55, bench.py:67
  * record parse ........... archive.py:233-275 (layout doc archive.py:1-30)
  * materialize (dequant) .. archive.py:278-325 (integer dequant archive.py:294-301)
  * CRC + reader ........... archive.py:328-400
  * PSNR ................... metrics.py:23-41 (+ u8 path image.py:49-55)
  * prune_l1 ............... compressor.py:100-152
  * quantize / codes ....... compressor.py:160-218
  * init / loss_and_grad ... net.py:152-171, 217-265
  * Adam / cosine / _train . net.py:268-300, encoder.py:28-30, 66-85
and one operation the reference does not have (SPEC.md:8 puts augmentation
out of scope), defined by this repo and pinned here so the GPU epilogue has a
checker: ``augment_coords`` / ``epilogue`` (crop / flip / normalise).
"""

from __future__ import annotations

import math
import struct
import zlib
from dataclasses import dataclass

import numpy as np

# archive.py:45-58 — container constants
MAGIC = b"RINR"
FORMAT_VERSION = 1
TAG_F32, TAG_F16, TAG_A8, TAG_A16 = range(4)
FORM_DENSE, FORM_DENSE_MASK, FORM_SPARSE = range(3)
QUANT_MODES = ("none", "affine8", "affine16")
_STORED_DTYPE = {TAG_F32: np.dtype("<f4"), TAG_F16: np.dtype("<f2"),
                 TAG_A8: np.dtype("<u1"), TAG_A16: np.dtype("<u2")}


class OracleIntegrityError(Exception):
    """Stand-in for rinr.errors.IntegrityError (errors.py:36-41)."""


# ----------------------------------------------------------------------------
# Model value types (net.py:24-118 reduced to what decode needs)
# ----------------------------------------------------------------------------

@dataclass
class OLayer:
    w: np.ndarray      # (out, in) f32 (f16 for TAG_F16 layers, net.py:196-197 upcasts)
    b: np.ndarray      # (out,) f32
    mask: np.ndarray   # (out, in) bool


@dataclass
class OModel:
    dims: tuple
    omega: float       # a Python float: keeps the forward in f32 (NEP 50)
    layers: list
    source_h: int = 0
    source_w: int = 0
    quant_mode: str = "none"
    quant: dict = None  # layer -> (bits, scale, zero_point, constant)


# ----------------------------------------------------------------------------
# Forward path
# ----------------------------------------------------------------------------

def coordinate_grid(h: int, w: int) -> np.ndarray:
    """(h*w, 2) f32 grid, x = c/(w-1), y = r/(h-1), 1-px axes map to 0.
    Same f64 linspace -> meshgrid -> f32 cast as net.py:146-149."""
    if h < 1 or w < 1:
        raise ValueError(f"grid dimensions must be >= 1, got {h}x{w}")
    axis_x = np.linspace(0.0, 1.0, w, dtype=np.float64) if w > 1 else np.zeros(1)
    axis_y = np.linspace(0.0, 1.0, h, dtype=np.float64) if h > 1 else np.zeros(1)
    x = np.broadcast_to(axis_x[None, :], (h, w)).reshape(-1)
    y = np.broadcast_to(axis_y[:, None], (h, w)).reshape(-1)
    return np.stack([x, y], axis=1).astype(np.float32)


def axis_coords(n: int) -> np.ndarray:
    """One axis of ``coordinate_grid`` as f32 (net.py:146-147)."""
    if n > 1:
        return np.linspace(0.0, 1.0, n, dtype=np.float64).astype(np.float32)
    return np.zeros(1, dtype=np.float32)


def forward(model: OModel, coords: np.ndarray) -> np.ndarray:
    """Raw (n, 3) network output.  Per layer ``z = a @ w.T + b`` in the
    activation dtype, hidden layers ``a = sin(omega * z)``, last layer affine
    (net.py:190-201)."""
    act = coords
    n_layers = len(model.layers)
    for li, layer in enumerate(model.layers):
        w = layer.w.astype(act.dtype) if layer.w.dtype != act.dtype else layer.w
        b = layer.b.astype(act.dtype) if layer.b.dtype != act.dtype else layer.b
        z = act @ w.T + b
        act = z if li == n_layers - 1 else np.sin(model.omega * z)
    return act


def decode(model: OModel, out_h=None, out_w=None) -> np.ndarray:
    """(h, w, 3) f32 in [0, 1] (decoder.py:19-36).  Quantised models carry
    already-dequantised weights, so dequantize() is the identity here."""
    h = model.source_h if out_h is None else out_h
    w = model.source_w if out_w is None else out_w
    if h < 1 or w < 1:
        raise ValueError(f"output size must be >= 1x1, got {h}x{w}")
    rgb = forward(model, coordinate_grid(h, w))
    return np.clip(rgb, 0.0, 1.0).reshape(h, w, 3)


def decode_batch(models, out_h=None, out_w=None):
    """Order-preserving list of decodes (decoder.py:39-61, parallelism=1)."""
    if not models:
        raise ValueError("empty model slice")
    return [decode(m, out_h, out_w) for m in models]


def to_u8(pixels: np.ndarray) -> np.ndarray:
    """floor(clip(v)*255 + 0.5) in f32 (image.py:49-55, bench.py:67)."""
    v = np.clip(pixels, 0.0, 1.0)
    return np.floor(v * np.float32(255.0) + np.float32(0.5)).astype(np.uint8)


def psnr(a: np.ndarray, b: np.ndarray, quantized: bool = False) -> float:
    """PSNR with peak 1.0 over normalised floats (metrics.py:23-41); the
    quantized variant goes through image.as_u8 (image.py:49-55) first."""
    if quantized:
        pa = to_u8(a).astype(np.float64) / 255.0
        pb = to_u8(b).astype(np.float64) / 255.0
    else:
        pa, pb = a.astype(np.float64), b.astype(np.float64)
    mse = float(np.mean((pa - pb) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)


# ----------------------------------------------------------------------------
# Augmentation epilogue (NOT in the reference: SPEC.md:8).  Defined by this
# repo; the CUDA epilogue implements exactly this arithmetic.
# ----------------------------------------------------------------------------

AUG_NONE, AUG_OFFSET, AUG_CROP = 0, 1, 2


def augment_coords(h: int, w: int, mode: int, params) -> tuple:
    """Source coordinates (n, 2) f32 and a validity mask for an h x w output.

    mode AUG_OFFSET, params (dx, dy, flip, pad): output column c reads source
      column j = (w-1-c if flip else c) + dx - pad (rows: r + dy - pad); the
      coordinate is the grid value of j, and j outside [0, w) is padding.
    mode AUG_CROP, params (x0, y0, sx, sy, flip): x = x0 + sx * gx[c'] with
      c' = w-1-c if flip else c, y = y0 + sy * gy[r], all f32 (mul then add,
      no fused multiply-add); every pixel is valid.
    """
    gx, gy = axis_coords(w), axis_coords(h)
    cols = np.arange(w)
    rows = np.arange(h)
    if mode == AUG_NONE:
        xs, ys = gx[cols], gy[rows]
        vx, vy = np.ones(w, bool), np.ones(h, bool)
    elif mode == AUG_OFFSET:
        dx, dy, flip, pad = (int(params[0]), int(params[1]), int(params[2]), int(params[3]))
        src_c = (w - 1 - cols if flip else cols) + dx - pad
        src_r = rows + dy - pad
        vx = (src_c >= 0) & (src_c < w)
        vy = (src_r >= 0) & (src_r < h)
        xs = np.where(vx, gx[np.clip(src_c, 0, w - 1)], np.float32(0))
        ys = np.where(vy, gy[np.clip(src_r, 0, h - 1)], np.float32(0))
    elif mode == AUG_CROP:
        x0, y0, sx, sy = (np.float32(v) for v in params[:4])
        flip = int(params[4])
        cx = w - 1 - cols if flip else cols
        xs = (sx * gx[cx]).astype(np.float32) + x0
        ys = (sy * gy[rows]).astype(np.float32) + y0
        vx, vy = np.ones(w, bool), np.ones(h, bool)
    else:
        raise ValueError(f"unknown augmentation mode {mode}")
    coords = np.stack([np.broadcast_to(xs[None, :], (h, w)).reshape(-1),
                       np.broadcast_to(ys[:, None], (h, w)).reshape(-1)], axis=1)
    valid = (vy[:, None] & vx[None, :]).reshape(-1)
    return coords.astype(np.float32), valid


def epilogue(raw: np.ndarray, valid: np.ndarray, h: int, w: int, mean, std) -> np.ndarray:
    """clamp -> zero-fill padding -> (v - mean)/std per channel, f32 CHW."""
    v = np.clip(raw, 0.0, 1.0).astype(np.float32)
    v[~valid] = 0.0
    m = np.asarray(mean, np.float32)
    s = np.asarray(std, np.float32)
    v = (v - m) / s
    return np.ascontiguousarray(v.reshape(h, w, 3).transpose(2, 0, 1))


def decode_augmented(model: OModel, h: int, w: int, mode: int, params, mean, std) -> np.ndarray:
    coords, valid = augment_coords(h, w, mode, params)
    return epilogue(forward(model, coords), valid, h, w, mean, std)


# ----------------------------------------------------------------------------
# .rinr container (archive.py)
# ----------------------------------------------------------------------------

class _Reader:
    """Bounds-checked little-endian cursor (archive.py:187-203)."""

    def __init__(self, buf: bytes, where: str):
        self.buf, self.pos, self.where = buf, 0, where

    def bytes(self, n: int) -> bytes:
        end = self.pos + n
        if end > len(self.buf):
            raise OracleIntegrityError(f"{self.where}: truncated (needed {n} bytes at {self.pos})")
        out = self.buf[self.pos:end]
        self.pos = end
        return out

    def fmt(self, f: str):
        return struct.unpack(f, self.bytes(struct.calcsize(f)))


@dataclass
class ORawLayer:
    tag: int
    form: int
    const: bool
    scale: float
    zero_point: int
    bitset: bytes | None
    values: np.ndarray
    bias: np.ndarray
    shape: tuple


@dataclass
class ORawRecord:
    rid: str
    source_h: int
    source_w: int
    dims: tuple
    omega: float
    quant_mode: str
    layers: list


def parse_record(body: bytes, where: str = "record") -> ORawRecord:
    """Record body (no CRC) -> raw sections (archive.py:233-275)."""
    rd = _Reader(body, where)
    (id_len,) = rd.fmt("<H")
    rid = rd.bytes(id_len).decode("utf-8")
    sh, sw = rd.fmt("<II")
    (nd,) = rd.fmt("<H")
    dims = rd.fmt(f"<{nd}H")
    (omega,) = rd.fmt("<d")
    if nd < 2 or dims[0] != 2 or dims[-1] != 3 or min(dims) < 1 or not omega > 0:
        raise OracleIntegrityError(f"{where}: bad architecture {dims} omega={omega}")
    (mode,) = rd.fmt("<B")
    if mode >= len(QUANT_MODES):
        raise OracleIntegrityError(f"{where}: unknown quant mode {mode}")
    layers = []
    for li in range(nd - 1):
        fan_in, fan_out = dims[li], dims[li + 1]
        n = fan_in * fan_out
        tag, form, const = rd.fmt("<BBB")
        if tag not in _STORED_DTYPE or form > FORM_SPARSE:
            raise OracleIntegrityError(f"{where}: layer {li} has bad tag/form {tag}/{form}")
        scale, zp = 1.0, 0
        if tag in (TAG_A8, TAG_A16):
            scale, zp = rd.fmt("<di")
        bitset = rd.bytes((n + 7) // 8) if form != FORM_DENSE else None
        kept = n
        if form == FORM_SPARSE:
            kept = int(np.unpackbits(np.frombuffer(bitset, np.uint8), count=n, bitorder="little").sum())
        dt = np.dtype("<f4") if (const and tag in (TAG_A8, TAG_A16)) else _STORED_DTYPE[tag]
        values = np.frombuffer(rd.bytes(kept * dt.itemsize), dtype=dt)
        bias = np.frombuffer(rd.bytes(4 * fan_out), dtype="<f4")
        layers.append(ORawLayer(tag, form, bool(const), scale, zp, bitset, values, bias, (fan_out, fan_in)))
    if rd.pos != len(body):
        raise OracleIntegrityError(f"{where}: {len(body) - rd.pos} trailing bytes")
    return ORawRecord(rid, sh, sw, tuple(dims), omega, QUANT_MODES[mode], layers)


def materialize(raw: ORawRecord) -> OModel:
    """Raw sections -> dense weights.  Affine codes: ``f32(f64 scale * (f64
    code - zp))`` with masked entries +0.0 (archive.py:294-301); float layers:
    zero-init then scatter/copy (archive.py:302-308)."""
    layers, quant = [], {}
    for li, rl in enumerate(raw.layers):
        n = rl.shape[0] * rl.shape[1]
        if rl.bitset is None:
            mask = np.ones(n, dtype=bool)
        else:
            mask = np.unpackbits(np.frombuffer(rl.bitset, np.uint8), count=n, bitorder="little").astype(bool)
        is_affine = rl.tag in (TAG_A8, TAG_A16)
        if is_affine and not rl.const:
            codes = np.zeros(n, dtype=np.float64)
            if rl.form == FORM_SPARSE:
                codes[mask] = rl.values.astype(np.float64)
            else:
                codes[:] = rl.values.astype(np.float64)
            w = (rl.scale * (codes - rl.zero_point)).astype(np.float32)
            w[~mask] = 0.0
        else:
            w = np.zeros(n, dtype=np.float16 if rl.tag == TAG_F16 else np.float32)
            if rl.form == FORM_SPARSE:
                w[mask] = rl.values
            else:
                w[:] = rl.values
        if is_affine:
            quant[li] = (8 if rl.tag == TAG_A8 else 16, rl.scale, rl.zero_point, rl.const)
        layers.append(OLayer(w.reshape(rl.shape), rl.bias.astype(np.float32).copy(), mask.reshape(rl.shape)))
    return OModel(raw.dims, raw.omega, layers, raw.source_h, raw.source_w, raw.quant_mode,
                  quant if raw.quant_mode != "none" else None)


def check_crc(blob: bytes, where: str) -> bytes:
    """Strip and verify the trailing CRC32 (archive.py:328-335)."""
    if len(blob) < 4:
        raise OracleIntegrityError(f"{where}: record too short for CRC")
    body = blob[:-4]
    (stored,) = struct.unpack("<I", blob[-4:])
    if zlib.crc32(body) & 0xFFFFFFFF != stored:
        raise OracleIntegrityError(f"{where}: CRC mismatch")
    return body


def record_blobs(data: bytes) -> list:
    """Header + chained index -> per-record byte ranges (archive.py:342-379)."""
    if len(data) < 10:
        raise OracleIntegrityError("truncated header")
    magic, version, count = struct.unpack_from("<4sHI", data, 0)
    if magic != MAGIC:
        raise OracleIntegrityError(f"bad magic {magic!r}")
    if version > FORMAT_VERSION:
        raise OracleIntegrityError(f"unsupported version {version}")
    if len(data) < 10 + 12 * count:
        raise OracleIntegrityError("truncated index")
    expect = 10 + 12 * count
    out = []
    for k in range(count):
        off, length = struct.unpack_from("<QI", data, 10 + 12 * k)
        if off != expect:
            raise OracleIntegrityError(f"record {k}: offset {off} != expected {expect}")
        expect = off + length
        blob = data[off:off + length]
        if len(blob) < length:
            raise OracleIntegrityError(f"record {k}: truncated body")
        out.append(blob)
    return out


def read_models(data: bytes) -> list:
    """Whole archive -> materialised models, validating every record
    (archive.py:395-400)."""
    return [materialize(parse_record(check_crc(b, f"record {k}"), f"record {k}"))
            for k, b in enumerate(record_blobs(data))]


def flat_params(model: OModel) -> np.ndarray:
    """[w0, b0, w1, b1, ...] as f32 — the layout ``rinr_dequantize`` writes."""
    parts = []
    for layer in model.layers:
        parts.append(layer.w.astype(np.float32).ravel())
        parts.append(layer.b.astype(np.float32).ravel())
    return np.concatenate(parts)


# ----------------------------------------------------------------------------
# Encoder-side transforms (checker for csrc/transforms.cu).
# ----------------------------------------------------------------------------

class OracleStructuralError(ValueError):
    """compressor.py:135-137 / 148-149 StructuralError."""


def prune_l1(weights: list, masks: list, total_ratio: float, scope: str = "global"):
    """compressor.py:108-152 on one model given as per-matrix (out, in) f32
    weights and bool masks; returns (weights, masks) copies."""
    if not (0.0 <= total_ratio < 1.0):
        raise ValueError("total_ratio must be in [0, 1)")
    w = [x.copy() for x in weights]
    m = [x.copy() for x in masks]
    if scope == "global":
        mags = np.concatenate([np.abs(x.ravel()).astype(np.float64) for x in weights])   # 102-104
        order = np.argsort(mags, kind="stable")
        k = int(math.floor(total_ratio * mags.size + 0.5))                               # 124
        flat = np.concatenate([x.ravel() for x in m]).copy()
        flat[order[:k]] = False
        off = 0
        for i in range(len(w)):
            sz = m[i].size
            new = flat[off:off + sz].reshape(m[i].shape) & m[i]
            off += sz
            if not new.any():
                raise OracleStructuralError("ratio would zero an entire layer")
            m[i] = new
            w[i] = np.multiply(w[i], new)                                                 # 138
    else:
        for i in range(len(w)):                                                           # 140-151
            mags = np.abs(w[i].ravel()).astype(np.float64)
            k = int(math.floor(total_ratio * mags.size + 0.5))
            new = m[i].ravel().copy()
            new[np.argsort(mags, kind="stable")[:k]] = False
            new = new.reshape(m[i].shape)
            if not new.any():
                raise OracleStructuralError("ratio would zero an entire layer")
            m[i] = new
            w[i] = np.multiply(w[i], new)
    return w, m


def quantize(weights: list, masks: list, biases: list, bits: int):
    """compressor.py:160-202: hidden matrices 1..L-2 snapped to the affine
    grid; returns (weights, {layer: (scale, zero_point, constant)})."""
    for x, b in zip(weights, biases):
        if not (np.isfinite(x).all() and np.isfinite(b).all()):
            raise ArithmeticError("non-finite weights")                                  # 172-174
    qmax = (1 << bits) - 1
    w = [x.copy() for x in weights]
    info = {}
    for i in range(1, len(w) - 1):
        kept = w[i][masks[i]].astype(np.float64)
        if kept.size == 0:
            info[i] = (1.0, 0, True)
            continue
        mn, mx = float(kept.min()), float(kept.max())
        if mx == mn:
            info[i] = (1.0, 0, True)
            continue
        scale = (mx - mn) / qmax
        zp = int(np.round(-mn / scale))
        if not (-(1 << 31) <= zp < (1 << 31)):
            info[i] = (1.0, 0, True)
            continue
        codes = np.clip(np.round(w[i].astype(np.float64) / scale) + zp, 0, qmax)
        snapped = (scale * (codes - zp)).astype(w[i].dtype)
        np.multiply(snapped, masks[i], out=snapped)
        w[i] = snapped
        info[i] = (scale, zp, False)
    return w, info


def quantize_codes(w: np.ndarray, scale: float, zp: int, bits: int) -> np.ndarray:
    """compressor.py:205-218 (codes recomputed from the snapped weights)."""
    qmax = (1 << bits) - 1
    codes = np.clip(np.round(w.astype(np.float64) / scale) + zp, 0, qmax)
    return codes.astype(np.uint8 if bits == 8 else np.uint16)


# ----------------------------------------------------------------------------
# Training (checker for the GPU encoder, csrc/fit.cu).  Models here are plain
# lists of per-layer f32 arrays: ws[l] (out, in), bs[l] (out,), ms[l] bool.
# ----------------------------------------------------------------------------

def init_model(dims, seed: int, omega: float = 30.0):
    """net.init (net.py:152-171): PCG64; layer 0 U(+-1/in), later
    U(+-sqrt(6/in)/omega), zero biases, all-ones masks."""
    rng = np.random.default_rng(seed)
    ws, bs, ms = [], [], []
    for li, (fi, fo) in enumerate(zip(dims[:-1], dims[1:])):
        bound = 1.0 / fi if li == 0 else np.sqrt(6.0 / fi) / omega
        ws.append(rng.uniform(-bound, bound, size=(fo, fi)).astype(np.float32))
        bs.append(np.zeros(fo, np.float32))
        ms.append(np.ones((fo, fi), bool))
    return ws, bs, ms


def loss_and_grad(ws, bs, ms, omega: float, coords, targets):
    """net.py:217-265 with reduction="mean": MSE over the 3n values and
    analytic gradients through the sine layers; masked gradient entries are 0."""
    a = coords
    zs, acts = [], [a]
    last = len(ws) - 1
    for i, (w, b) in enumerate(zip(ws, bs)):                                   # 183-202
        z = a @ w.T + b
        zs.append(z)
        a = z if i == last else np.sin(omega * z)
        acts.append(a)
    resid = acts[-1] - targets
    scale = 1.0 / resid.size
    loss = float((resid.astype(np.float64) ** 2).sum() * scale)
    gws, gbs = [None] * len(ws), [None] * len(ws)
    delta = (2.0 * scale) * resid
    for i in range(len(ws) - 1, -1, -1):                                       # 256-264
        gw = delta.T @ acts[i]
        gb = delta.sum(axis=0)
        np.multiply(gw, ms[i], out=gw)
        gws[i], gbs[i] = gw, gb
        if i > 0:
            delta = (delta @ ws[i]) * (omega * np.cos(omega * zs[i - 1]))
    return loss, gws, gbs


class Adam:
    """net.Adam (net.py:268-300): f32 moments, bias corrections from Python
    floats, mask re-applied after every step."""

    def __init__(self, ws, bs, beta1=0.9, beta2=0.999, eps=1e-8):
        self.beta1, self.beta2, self.eps, self.t = beta1, beta2, eps, 0
        self.m = [(np.zeros_like(w), np.zeros_like(b)) for w, b in zip(ws, bs)]
        self.v = [(np.zeros_like(w), np.zeros_like(b)) for w, b in zip(ws, bs)]

    def step(self, ws, bs, ms, gws, gbs, lr: float):
        self.t += 1
        c1 = 1.0 - self.beta1 ** self.t
        c2 = 1.0 - self.beta2 ** self.t
        for l in range(len(ws)):
            for j, (p, g) in enumerate(((ws[l], gws[l]), (bs[l], gbs[l]))):
                g = g.astype(p.dtype, copy=False)
                mp, vp = self.m[l][j], self.v[l][j]
                mp *= self.beta1
                mp += (1.0 - self.beta1) * g
                vp *= self.beta2
                vp += (1.0 - self.beta2) * g * g
                p -= lr * (mp / c1) / (np.sqrt(vp / c2) + self.eps)
            np.multiply(ws[l], ms[l], out=ws[l])


def cosine_lr(lr0: float, t: int, total: int) -> float:
    """encoder.py:28-30."""
    return 0.5 * lr0 * (1.0 + math.cos(math.pi * t / total))


def train(ws, bs, ms, omega, coords, targets, lr0: float, steps: int):
    """encoder._train (encoder.py:66-85): full-batch Adam + cosine decay;
    returns the sampled loss curve (every max(1, steps // 64) steps + final)."""
    opt = Adam(ws, bs)
    stride = max(1, steps // 64)
    curve = []
    for t in range(steps):
        loss, gws, gbs = loss_and_grad(ws, bs, ms, omega, coords, targets)
        if not math.isfinite(loss):
            raise ArithmeticError(f"loss became non-finite at step {t}")
        if t % stride == 0:
            curve.append(loss)
        opt.step(ws, bs, ms, gws, gbs, cosine_lr(lr0, t, steps))
    loss, _, _ = loss_and_grad(ws, bs, ms, omega, coords, targets)
    curve.append(loss)
    return curve
