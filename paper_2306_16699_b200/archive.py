"""The .rinr container on the host: a vectorised writer and the record types.

Layout and writer rules are the reference's (archive.py:1-30, 92-184); the
writer here builds every record of a same-architecture batch with array
operations instead of a per-record loop (a 262k-record store is built in a
few seconds), and is byte-identical to the reference writer
(tests/test_archive_writer.py).  Reading/parsing is native: the C++ store
loader (csrc/store.cpp, ``Store``) validates header, index, CRC and every
record, and materialisation happens on the GPU inside each decode.
"""

from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .compressor import ModelBatch, quantize_codes_batch
from .errors import InvalidInputError
from .net import validate_model

MAGIC = b"RINR"
VERSION = 1
HEADER_FMT = "<4sHI"
HEADER_SIZE = struct.calcsize(HEADER_FMT)  # 10
INDEX_ENTRY_FMT = "<QI"
INDEX_ENTRY_SIZE = struct.calcsize(INDEX_ENTRY_FMT)  # 12

TAG_F32, TAG_F16, TAG_A8, TAG_A16 = 0, 1, 2, 3
FORM_DENSE, FORM_DENSE_MASK, FORM_SPARSE = 0, 1, 2
SPARSE_THRESHOLD = 0.125
_MODE_CODES = {"none": 0, "affine8": 1, "affine16": 2}


@dataclass
class ArchiveRecord:
    id: str
    model: object


@dataclass
class DatasetArchive:
    records: list = field(default_factory=list)
    version: int = VERSION

    def __post_init__(self):
        ids = [r.id for r in self.records]
        if len(set(ids)) != len(ids):
            raise InvalidInputError("record ids must be unique")

    def __len__(self) -> int:
        return len(self.records)

    def ids(self) -> list:
        return [r.id for r in self.records]


class _Field:
    """One variable-length byte field for every record: a left-packed
    [N, width] u8 matrix plus per-record byte counts."""

    __slots__ = ("mat", "lens")

    def __init__(self, mat: np.ndarray, lens: np.ndarray):
        self.mat = np.ascontiguousarray(mat, dtype=np.uint8)
        self.lens = np.asarray(lens, dtype=np.int64)


def _const_field(n: int, data: bytes) -> _Field:
    row = np.frombuffer(data, np.uint8)
    return _Field(np.broadcast_to(row, (n, row.size)), np.full(n, row.size))


def _packed_values(values: np.ndarray, select: np.ndarray) -> _Field:
    """Left-pack the selected elements of each row (row-major order kept) and
    view them as bytes: the 'values' section (archive.py:132-135)."""
    n, m = values.shape
    isz = values.dtype.itemsize
    if select.all():
        packed = values
        count = np.full(n, m)
    else:
        order = np.argsort(~select, axis=1, kind="stable")  # kept entries first, in order
        packed = np.take_along_axis(values, order, axis=1)
        count = select.sum(axis=1)
    return _Field(np.ascontiguousarray(packed).view(np.uint8).reshape(n, m * isz), count * isz)


def _layer_fields(mb: ModelBatch, l: int) -> list:
    n = mb.n
    w, b, mask = mb.w[l], mb.b[l], mb.mask[l]
    size = mask.shape[1] * mask.shape[2]
    mflat = mask.reshape(n, size)
    zeros = size - mflat.sum(axis=1)
    # form by zero fraction (archive.py:100-108)
    form = np.where(zeros == 0, FORM_DENSE, np.where(zeros / size > SPARSE_THRESHOLD, FORM_SPARSE, FORM_DENSE_MASK))
    q = mb.quant.get(l) if mb.quant_mode != "none" else None
    if q is not None:
        tag = TAG_A8 if q.bits == 8 else TAG_A16
        const = q.constant
    else:
        tag = TAG_F16 if w.dtype == np.float16 else TAG_F32
        const = np.zeros(n, bool)
    fields = [_Field(np.stack([np.full(n, tag), form, const.astype(np.int64)], axis=1), np.full(n, 3))]
    if q is not None:
        hdr = np.zeros((n, 12), np.uint8)
        hdr[:, :8] = q.scale.astype("<f8").view(np.uint8).reshape(n, 8)
        hdr[:, 8:] = q.zero_point.astype("<i4").view(np.uint8).reshape(n, 4)
        fields.append(_Field(hdr, np.full(n, 12)))
    bits = np.packbits(mflat, axis=1, bitorder="little")
    fields.append(_Field(bits, np.where(form != FORM_DENSE, bits.shape[1], 0)))
    select = mflat | (form != FORM_SPARSE)[:, None]
    float_vals = w.reshape(n, size).astype("<f2" if tag == TAG_F16 else "<f4")
    if q is not None and not const.all():
        codes = quantize_codes_batch(mb, l).astype("<u1" if q.bits == 8 else "<u2")
        fc = _packed_values(codes, select)
        if const.any():
            ff = _packed_values(float_vals, select)
            width = max(fc.mat.shape[1], ff.mat.shape[1])
            mat = np.zeros((n, width), np.uint8)
            mat[~const, :fc.mat.shape[1]] = fc.mat[~const]
            mat[const, :ff.mat.shape[1]] = ff.mat[const]
            fields.append(_Field(mat, np.where(const, ff.lens, fc.lens)))
        else:
            fields.append(fc)
    else:
        fields.append(_packed_values(float_vals, select))
    fields.append(_Field(b.astype("<f4").view(np.uint8).reshape(n, -1), np.full(n, b.shape[1] * 4)))
    return fields


def _assemble(fields: list, n: int) -> tuple:
    """Concatenate per-record fields into one buffer, leaving 4 bytes per
    record for the CRC.  Returns (buffer, record starts, record lengths)."""
    lens = np.stack([f.lens for f in fields], axis=1)  # [N, F]
    body = lens.sum(axis=1)
    rec_len = body + 4
    starts = np.concatenate([[0], np.cumsum(rec_len)[:-1]])
    field_start = starts[:, None] + np.concatenate([np.zeros((n, 1), np.int64), np.cumsum(lens, axis=1)[:, :-1]], 1)
    out = np.zeros(int(rec_len.sum()), np.uint8)
    for fi, f in enumerate(fields):
        width = f.mat.shape[1]
        if width == 0:
            continue
        dest = field_start[:, fi][:, None] + np.arange(width)[None, :]
        if bool((f.lens == width).all()):  # every record writes the full row: no compaction
            out[dest] = f.mat
            continue
        sel = np.arange(width)[None, :] < f.lens[:, None]
        out[dest[sel]] = f.mat[sel]
    return out, starts, body


def encode_batch(mb: ModelBatch, ids) -> list:
    """Record bodies (CRC included) for every record of the batch."""
    buf, starts, body = _encode_batch_buffer(mb, ids)
    return [bytes(buf[s:s + b + 4]) for s, b in zip(starts, body)]


def _encode_batch_buffer(mb: ModelBatch, ids) -> tuple:
    n = mb.n
    if len(ids) != n:
        raise InvalidInputError("one id per record required")
    dims = mb.arch.dims
    if max(dims) > 0xFFFF:
        raise InvalidInputError(f"layer widths above 65535 are not serializable: {dims}")
    id_bytes = [str(i).encode("utf-8") for i in ids]
    id_len = np.array([len(b) for b in id_bytes], np.int64)
    if id_len.max(initial=0) > 0xFFFF:
        raise InvalidInputError("record id longer than 65535 bytes")
    width = int(id_len.max(initial=0))
    id_mat = np.zeros((n, 2 + width), np.uint8)
    id_mat[:, :2] = id_len.astype("<u2").view(np.uint8).reshape(n, 2)
    if width:
        flat = np.frombuffer(b"".join(id_bytes), np.uint8)
        sel = np.arange(width)[None, :] < id_len[:, None]
        id_mat[:, 2:][sel] = flat
    fields = [_Field(id_mat, id_len + 2)]
    fields.append(_const_field(n, struct.pack("<II", mb.source_h, mb.source_w) +
                               struct.pack(f"<H{len(dims)}H", len(dims), *dims) +
                               struct.pack("<d", mb.arch.omega) +
                               struct.pack("<B", _MODE_CODES[mb.quant_mode])))
    for l in range(len(mb.w)):
        fields.extend(_layer_fields(mb, l))
    buf, starts, body = _assemble(fields, n)
    mv = memoryview(buf)
    crcs = np.fromiter((zlib.crc32(mv[s:s + b]) for s, b in zip(starts.tolist(), body.tolist())),
                       dtype="<u4", count=n)
    tails = (starts + body)[:, None] + np.arange(4)[None, :]
    buf[tails.ravel()] = crcs.view(np.uint8)
    return buf, starts, body


def serialize_batch(mb: ModelBatch, ids) -> bytes:
    """Whole-archive bytes for a same-architecture batch (archive.py:165-174)."""
    buf, starts, body = _encode_batch_buffer(mb, ids)
    return _wrap(buf, body + 4)


def _wrap(records: np.ndarray, lengths: np.ndarray) -> bytes:
    n = lengths.size
    first = HEADER_SIZE + INDEX_ENTRY_SIZE * n
    offs = first + np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    index = np.zeros(n, dtype=[("off", "<u8"), ("len", "<u4")])
    index["off"] = offs
    index["len"] = lengths
    return struct.pack(HEADER_FMT, MAGIC, VERSION, n) + index.tobytes() + records.tobytes()


def encode_record(record) -> bytes:
    """One record (ArchiveRecord with an InrModel) -> bytes incl. CRC
    (archive.py:140-158)."""
    validate_model(record.model)
    return encode_batch(ModelBatch.from_models([record.model]), [record.id])[0]


def serialize(archive) -> bytes:
    """Archive of arbitrary (possibly mixed-architecture) records."""
    bodies = [encode_record(r) for r in archive.records]
    lengths = np.array([len(b) for b in bodies], np.int64)
    return _wrap(np.frombuffer(b"".join(bodies), np.uint8), lengths)


def write(archive, sink) -> int:
    data = serialize(archive)
    if hasattr(sink, "write"):
        sink.write(data)
    else:
        Path(sink).write_bytes(data)
    return len(data)
