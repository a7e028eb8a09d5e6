"""read / ArchiveReader.read_record / materialize (reader.py) against the
reference's materialised models (golden 'params': archive.read in the
reference) and the oracle: weights bit-exact (uint32), masks, biases,
quantisation metadata, f16 layer dtypes; corrupt archives raise
IntegrityError naming the record."""

import numpy as np
import pytest

from conftest import STORE_CASES
from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu


def _same(model, om, flat_ref):
    flat = np.concatenate([np.concatenate([l.w.astype(np.float32).ravel(), l.b.ravel()]) for l in model.layers])
    np.testing.assert_array_equal(flat.view(np.uint32), flat_ref[:flat.size].view(np.uint32))
    for l, ol in zip(model.layers, om.layers):
        assert l.w.dtype == ol.w.dtype
    for m, ol in zip(model.mask, om.layers):
        np.testing.assert_array_equal(m, ol.mask)
    if om.quant is None:
        assert model.quant is None
    else:
        assert model.quant.mode == om.quant_mode
        for li, (bits, scale, zp, const) in om.quant.items():
            q = model.quant.layers[li]
            assert (q.bits, q.scale, q.zero_point, q.constant) == (bits, scale, zp, const)


@pytest.mark.parametrize("case", STORE_CASES)
def test_read_matches_reference(golden, case):
    from paper_2306_16699_b200 import ArchiveReader, materialize, read
    g = golden(case)
    data = g["archive"].tobytes()
    oms = O.read_models(data)
    ds = read(data)
    assert len(ds) == len(oms) and ds.version == 1
    for k, (rec, om) in enumerate(zip(ds.records, oms)):
        _same(rec.model, om, g["params"][k])
    rd = ArchiveReader(data)
    for k in (0, len(rd) - 1):
        rec = rd.read_record(k)
        assert rec.id == ds.records[k].id
        _same(rec.model, oms[k], g["params"][k])
        raw = rd.read_raw(k)
        raw.body = b""  # a hand-built RawRecord: re-encoded before the native path
        _same(materialize(raw).model, oms[k], g["params"][k])


def test_read_corrupt_names_record(golden):
    from paper_2306_16699_b200 import IntegrityError, read
    from paper_2306_16699_b200.reader import ArchiveReader
    data = bytearray(golden("c2")["archive"].tobytes())
    off, _ = ArchiveReader(bytes(data)).index[3]
    data[off + 9] ^= 0x5A
    with pytest.raises(IntegrityError) as e:
        read(bytes(data))
    assert "record 3" in str(e.value) or getattr(e.value, "record", None) == "record 3"


def test_read_then_decode_roundtrip(golden):
    """read() -> decode_batch(models): the reference's two-call workflow."""
    from paper_2306_16699_b200 import decode_batch, read
    g = golden("c2")
    ds = read(g["archive"].tobytes())
    imgs = decode_batch([r.model for r in ds.records], 32, 32)
    got = np.stack([im.pixels for im in imgs])
    assert float(np.abs(got - g["decode_32x32"]).max()) <= 1e-3
