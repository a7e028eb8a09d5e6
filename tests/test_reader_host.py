"""Host side of the reader drop-ins (reader.py; archive.py:186-382 of the
reference): parse_record against the oracle's parse on every golden archive,
ArchiveReader's header / index / CRC checks and error messages."""

import struct

import numpy as np
import pytest

from conftest import STORE_CASES
from oracle import rinr_oracle as O
from paper_2306_16699_b200 import reader as R
from paper_2306_16699_b200.errors import IntegrityError, InvalidInputError


@pytest.mark.parametrize("case", STORE_CASES + ["fitted"])
def test_parse_record_matches_oracle(golden, case):
    g = golden(case)
    keys = [k for k in g if k.endswith("archive")]
    for key in keys:
        data = g[key].tobytes()
        rd = R.ArchiveReader(data)
        blobs = O.record_blobs(data)
        assert len(rd) == len(blobs)
        for k, blob in enumerate(blobs):
            raw = rd.read_raw(k)
            want = O.parse_record(O.check_crc(blob, "r"), "r")
            assert (raw.id, raw.source_h, raw.source_w, raw.arch.dims, raw.arch.omega, raw.quant_mode) == \
                (want.rid, want.source_h, want.source_w, want.dims, want.omega, want.quant_mode)
            for a, b in zip(raw.layers, want.layers):
                assert (a.tag, a.form, a.const, a.zero_point, a.mask_bits, a.shape) == \
                    (b.tag, b.form, b.const, b.zero_point, b.bitset, b.shape)
                assert np.float64(a.scale).view(np.uint64) == np.float64(b.scale).view(np.uint64)
                np.testing.assert_array_equal(a.values, b.values)
                np.testing.assert_array_equal(a.bias.view(np.uint32), b.bias.view(np.uint32))
            assert R._reencode(raw) == raw.body  # hand-built records re-encode byte for byte


def test_reader_errors(golden):
    data = bytearray(golden("c2")["archive"].tobytes())
    rd = R.ArchiveReader(bytes(data))
    with pytest.raises(InvalidInputError, match="out of range"):
        rd.read_raw(len(rd))
    off, length = rd.index[2]
    bad = bytearray(data)
    bad[off + 5] ^= 0xFF
    rd2 = R.ArchiveReader(bytes(bad))  # open checks header + index only
    rd2.read_raw(1)
    with pytest.raises(IntegrityError, match="record 2: CRC mismatch"):
        rd2.read_raw(2)
    with pytest.raises(IntegrityError, match="bad magic"):
        R.ArchiveReader(b"XXXX" + bytes(data[4:]))
    with pytest.raises(IntegrityError, match="truncated header"):
        R.ArchiveReader(bytes(data[:6]))
    with pytest.raises(IntegrityError, match="truncated index"):
        R.ArchiveReader(bytes(data[:20]))
    chained = bytearray(data)
    struct.pack_into("<Q", chained, 10 + 12 * 1, rd.index[1][0] + 1)
    with pytest.raises(IntegrityError, match="record 1: offset"):
        R.ArchiveReader(bytes(chained))
    body = rd._body(0)
    with pytest.raises(IntegrityError, match="trailing bytes"):
        R.parse_record(body + b"\0", "record 0")
    with pytest.raises(IntegrityError, match="truncated"):
        R.parse_record(body[:-3], "record 0")
