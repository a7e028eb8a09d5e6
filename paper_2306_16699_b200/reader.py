"""Reader drop-ins of the reference archive API, backed by the native loader
and the GPU dequantisation:

  * ``parse_record(body)``  -> ``RawRecord``   (archive.py:206-275): host byte
    walk of one CRC-stripped record body, the reference's error messages;
  * ``materialize(raw)``    -> ``ArchiveRecord`` (archive.py:278-325): weights
    from ``rinr_dequantize`` (bit-exact with the reference, uint32 compares in
    the tests), masks from the kept bitsets, QuantInfo rebuilt;
  * ``ArchiveReader(source)`` (archive.py:328-382): header + chained index
    checked at open, random access ``read_raw(k)`` / ``read_record(k)`` with
    the per-record CRC;
  * ``read(source)``        -> ``DatasetArchive`` (archive.py:395-400): the
    whole archive validated by the C++ loader (header, index chain, CRC and
    parse of every record; IntegrityError naming the first bad record) and
    materialised by ONE dequantise launch over all records.

The model / record types are this package's (duck-compatible with rinr's);
``decoder.install()`` switches them to the reference's own classes.
"""

from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import archive as A
from .compressor import LayerQuant, QuantInfo
from .errors import IntegrityError, InvalidInputError
from .net import Architecture, InrModel, LayerWeights, validate_model

_DTYPE_OF_TAG = {A.TAG_F32: np.dtype("<f4"), A.TAG_F16: np.dtype("<f2"), A.TAG_A8: np.dtype("<u1"),
                 A.TAG_A16: np.dtype("<u2")}
_MODE_NAMES = {0: "none", 1: "affine8", 2: "affine16"}

# classes the materialised objects are built from (install() rebinds them)
TYPES = {"InrModel": InrModel, "LayerWeights": LayerWeights, "QuantInfo": QuantInfo, "LayerQuant": LayerQuant,
         "Architecture": Architecture, "ArchiveRecord": A.ArchiveRecord, "DatasetArchive": A.DatasetArchive}


@dataclass
class RawLayer:
    """One stored layer before dequantisation (archive.py:206-218)."""

    tag: int
    form: int
    const: bool
    scale: float
    zero_point: int
    mask_bits: bytes | None
    values: np.ndarray
    bias: np.ndarray
    shape: tuple


@dataclass
class RawRecord:
    """A parsed, not yet materialised record (archive.py:221-230)."""

    id: str
    source_h: int
    source_w: int
    arch: object
    quant_mode: str
    layers: list
    body: bytes = field(default=b"", repr=False)  # the CRC-stripped bytes (native materialise)


def parse_record(body: bytes, context: str = "record") -> RawRecord:
    """Walk one record body (CRC already checked)."""
    buf = memoryview(bytes(body))
    end = len(buf)
    pos = 0

    def need(n):
        nonlocal pos
        if pos + n > end:
            raise IntegrityError(f"{context}: truncated (needed {n} bytes at {pos})")
        at = pos
        pos += n
        return at

    id_len = struct.unpack_from("<H", buf, need(2))[0]
    rid = bytes(buf[need(id_len):pos]).decode("utf-8")
    source_h, source_w = struct.unpack_from("<II", buf, need(8))
    nd = struct.unpack_from("<H", buf, need(2))[0]
    dims = struct.unpack_from(f"<{nd}H", buf, need(2 * nd))
    omega = struct.unpack_from("<d", buf, need(8))[0]
    try:
        arch = TYPES["Architecture"](dims, omega)
    except InvalidInputError as e:
        raise IntegrityError(f"{context}: bad architecture: {e}") from e
    mode = buf[need(1)]
    if mode not in _MODE_NAMES:
        raise IntegrityError(f"{context}: unknown quant mode {mode}")
    layers = []
    for li in range(len(dims) - 1):
        fi, fo = dims[li], dims[li + 1]
        n = fi * fo
        at = need(3)
        tag, form, cst = buf[at], buf[at + 1], buf[at + 2]
        if tag not in _DTYPE_OF_TAG or form > A.FORM_SPARSE:
            raise IntegrityError(f"{context}: layer {li} has bad tag/form {tag}/{form}")
        affine = tag in (A.TAG_A8, A.TAG_A16)
        scale, zp = struct.unpack_from("<di", buf, need(12)) if affine else (1.0, 0)
        bits = bytes(buf[need((n + 7) // 8):pos]) if form != A.FORM_DENSE else None
        kept = n
        if form == A.FORM_SPARSE:
            kept = int(np.unpackbits(np.frombuffer(bits, np.uint8), count=n, bitorder="little").sum())
        dt = np.dtype("<f4") if (cst and affine) else _DTYPE_OF_TAG[tag]
        values = np.frombuffer(buf, dt, count=kept, offset=need(kept * dt.itemsize))
        bias = np.frombuffer(buf, "<f4", count=fo, offset=need(4 * fo))
        layers.append(RawLayer(tag, form, bool(cst), scale, zp, bits, values, bias, (fo, fi)))
    if pos != end:
        raise IntegrityError(f"{context}: {end - pos} trailing bytes")
    return RawRecord(rid, source_h, source_w, arch, _MODE_NAMES[mode], layers, bytes(buf))


def _model(raw: RawRecord, flat: np.ndarray):
    """InrModel of a parsed record from its dequantised flat parameters
    [w0, b0, w1, b1, ...] (rinr_dequantize layout)."""
    T = TYPES
    layers, masks, qlayers = [], [], {}
    off = 0
    for li, rl in enumerate(raw.layers):
        fo, fi = rl.shape
        n = fo * fi
        w = flat[off:off + n].reshape(fo, fi)
        off += n + fo
        if rl.tag == A.TAG_F16:
            w = w.astype(np.float16)  # exact: the f16 values were widened on the GPU
        mask = (np.unpackbits(np.frombuffer(rl.mask_bits, np.uint8), count=n, bitorder="little").astype(bool)
                if rl.mask_bits is not None else np.ones(n, bool)).reshape(fo, fi)
        layers.append(T["LayerWeights"](np.ascontiguousarray(w), rl.bias.astype(np.float32).copy()))
        masks.append(mask)
        if rl.tag in (A.TAG_A8, A.TAG_A16):
            qlayers[li] = T["LayerQuant"](8 if rl.tag == A.TAG_A8 else 16, rl.scale, rl.zero_point, rl.const)
    quant = T["QuantInfo"](raw.quant_mode, qlayers) if raw.quant_mode != "none" else None
    model = T["InrModel"](arch=raw.arch, layers=layers, mask=masks, source_h=raw.source_h, source_w=raw.source_w,
                          quant=quant)
    validate_model(model)
    return model


def _dequantize_all(data: bytes, n: int) -> np.ndarray:
    import torch  # noqa: PLC0415

    from .store import Store  # noqa: PLC0415
    with Store(data) as st:  # native validation of every record (IntegrityError naming it)
        return st.dequantize(torch.arange(n)).cpu().numpy()


def materialize(raw: RawRecord):
    """archive.materialize: dequantised weights from the GPU kernel."""
    body = raw.body or _reencode(raw)
    rec = body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)
    flat = _dequantize_all(A._wrap(np.frombuffer(rec, np.uint8), np.array([len(rec)])), 1)[0]
    return TYPES["ArchiveRecord"](raw.id, _model(raw, flat))


def _reencode(raw: RawRecord) -> bytes:
    """Body bytes of a RawRecord built by hand (no stored body)."""
    dims = raw.arch.dims
    mode = {v: k for k, v in _MODE_NAMES.items()}[raw.quant_mode]
    rid = raw.id.encode("utf-8")
    out = [struct.pack("<H", len(rid)), rid, struct.pack("<II", raw.source_h, raw.source_w),
           struct.pack(f"<H{len(dims)}H", len(dims), *dims), struct.pack("<d", raw.arch.omega), bytes([mode])]
    for rl in raw.layers:
        out.append(bytes([rl.tag, rl.form, int(rl.const)]))
        if rl.tag in (A.TAG_A8, A.TAG_A16):
            out.append(struct.pack("<di", rl.scale, rl.zero_point))
        if rl.form != A.FORM_DENSE:
            out.append(rl.mask_bits)
        out.append(np.ascontiguousarray(rl.values).tobytes())
        out.append(np.ascontiguousarray(rl.bias, "<f4").tobytes())
    return b"".join(out)


def _source_bytes(source) -> bytes:
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    if hasattr(source, "read"):
        return source.read()
    return Path(source).read_bytes()


class ArchiveReader:
    """Random access over an archive (archive.py:328-382): the header and the
    chained index are checked at open, record k's CRC when it is read."""

    def __init__(self, source):
        self._data = _source_bytes(source)
        d = self._data
        if len(d) < A.HEADER_SIZE:
            raise IntegrityError("truncated header")
        magic, version, count = struct.unpack_from(A.HEADER_FMT, d, 0)
        if magic != A.MAGIC:
            raise IntegrityError(f"bad magic {magic!r}")
        if version > A.VERSION:
            raise IntegrityError(f"unsupported version {version}")
        self.version = version
        if len(d) < A.HEADER_SIZE + A.INDEX_ENTRY_SIZE * count:
            raise IntegrityError("truncated index")
        idx = np.frombuffer(d, np.dtype([("off", "<u8"), ("len", "<u4")]), count=count, offset=A.HEADER_SIZE)
        self.index = [(int(o), int(n)) for o, n in zip(idx["off"], idx["len"])]
        expect = A.HEADER_SIZE + A.INDEX_ENTRY_SIZE * count
        for k, (off, length) in enumerate(self.index):
            if off != expect:
                raise IntegrityError(f"record {k}: offset {off} != expected {expect}")
            expect = off + length

    def __len__(self) -> int:
        return len(self.index)

    def _body(self, k: int) -> bytes:
        if not (0 <= k < len(self.index)):
            raise InvalidInputError(f"record {k} out of range [0, {len(self.index)})")
        off, length = self.index[k]
        blob = self._data[off:off + length]
        if len(blob) < length:
            raise IntegrityError(f"record {k}: truncated body")
        if length < 4:
            raise IntegrityError(f"record {k}: record too short for CRC")
        body, stored = blob[:-4], struct.unpack("<I", blob[-4:])[0]
        actual = zlib.crc32(body) & 0xFFFFFFFF
        if stored != actual:
            raise IntegrityError(f"record {k}: CRC mismatch (stored {stored:#010x}, computed {actual:#010x})")
        return body

    def read_raw(self, k: int) -> RawRecord:
        return parse_record(self._body(k), f"record {k}")

    def read_record(self, k: int):
        return materialize(self.read_raw(k))

    def close(self) -> None:
        self._data = b""

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def read(source):
    """archive.read: load and fully validate an archive; nothing partial is
    returned.  One native parse + one GPU dequantise for all records."""
    data = _source_bytes(source)
    reader = ArchiveReader(data)
    n = len(reader)
    flat = _dequantize_all(data, n) if n else np.zeros((0, 0), np.float32)
    records = []
    for k in range(n):
        off, length = reader.index[k]
        raw = parse_record(data[off:off + length - 4], f"record {k}")
        records.append(TYPES["ArchiveRecord"](raw.id, _model(raw, flat[k])))
    return TYPES["DatasetArchive"](records=records, version=reader.version)
