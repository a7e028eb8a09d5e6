"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host parser (csrc/store.cpp) accepts/rejects exactly
what the reference reader does (archive.py:338-400) — no GPU needed."""

import ctypes
import re
import struct

import numpy as np
import pytest

from conftest import ROOT, STORE_CASES
from oracle import rinr_oracle as O
from paper_2306_16699_b200 import _native as N
from paper_2306_16699_b200 import errors


def header_symbols(names=("rinr_b200.h", "rinr_b200_transforms.h", "rinr_b200_encoder.h", "rinr_b200_writer.h")):
    text = "".join((ROOT / "include" / h).read_text() for h in names)
    return sorted(set(re.findall(r"RINR_API\s+[\w\s\*]+?\b(rinr_\w+)\s*\(", text)))


def test_library_exports_header_symbols():
    lib = N.lib()
    syms = header_symbols()
    assert set(syms) == set(N.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.rinr_abi_version() == 1
    for s in header_symbols(("rinr_b200_diag.h",)):
        assert hasattr(lib, s), s


def test_header_constants_match_python_mirror():
    """The enum / flag #defines of rinr_b200.h and the ctypes mirror agree."""
    text = (ROOT / "include" / "rinr_b200.h").read_text()
    defs = {k: int(v) for k, v in re.findall(r"#define\s+RINR_(\w+)\s+(-?\d+)\b", text)}
    for name in ("FLAG_OVERLAP_PROLOGUE", "FLAG_PREFETCH_NEXT"):
        assert defs[name] == getattr(N, name), name
    assert defs["FLAG_OVERLAP_PROLOGUE"] & defs["FLAG_PREFETCH_NEXT"] == 0


@pytest.mark.parametrize("case", STORE_CASES)
def test_validate_golden(golden, case):
    data = golden(case)["archive"].tobytes()
    assert N.archive_validate(data) == len(O.record_blobs(data))


def _corruptions(data: bytes):
    n = struct.unpack_from("<I", data, 6)[0]
    off1, len1 = struct.unpack_from("<QI", data, 10 + 12)
    yield "truncated header", data[:7]
    yield "bad magic", b"RINX" + data[4:]
    yield "unsupported version", data[:4] + struct.pack("<H", 2) + data[6:]
    yield "truncated index", data[:10 + 12 * n - 1]
    b = bytearray(data)
    struct.pack_into("<Q", b, 10 + 12, off1 + 1)
    yield "record 1: offset", bytes(b)
    b = bytearray(data)
    b[off1 + 20] ^= 0x40
    yield "record 1: CRC mismatch", bytes(b)
    yield f"record {n - 1}: truncated body", data[:-3]
    # a structurally bad record with a valid CRC: unknown quant mode
    import zlib
    body = bytearray(data[off1:off1 + len1 - 4])
    idlen = struct.unpack_from("<H", body, 0)[0]
    nd = struct.unpack_from("<H", body, 2 + idlen + 8)[0]
    body[2 + idlen + 8 + 2 + 2 * nd + 8] = 7
    b = bytearray(data)
    b[off1:off1 + len1] = bytes(body) + struct.pack("<I", zlib.crc32(bytes(body)))
    yield "record 1: unknown quant mode", bytes(b)


@pytest.mark.parametrize("case", ["c1_r1", "c2", "zoo"])
def test_integrity_errors_match_oracle(golden, case):
    data = golden(case)["archive"].tobytes()
    for what, bad in _corruptions(data):
        with pytest.raises(O.OracleIntegrityError) as ref:
            O.read_models(bad)
        with pytest.raises(errors.IntegrityError) as got:
            N.archive_validate(bad)
        assert what in str(got.value), (what, str(got.value))
        assert str(ref.value).split(":")[0] == str(got.value).split(":")[0]


def test_duplicate_ids_rejected(golden):
    from paper_2306_16699_b200 import synth
    from paper_2306_16699_b200.archive import serialize_batch
    mb = synth.seeded_batch(synth.ARCH_A, range(3))
    data = serialize_batch(mb, ["a", "b", "a"])
    with pytest.raises(errors.InvalidInputError, match="unique"):
        N.archive_validate(data)


def test_empty_archive():
    from paper_2306_16699_b200.archive import _wrap
    data = _wrap(np.zeros(0, np.uint8), np.zeros(0, np.int64))
    assert N.archive_validate(data) == 0


def test_error_is_thread_local():
    lib = N.lib()
    with pytest.raises(errors.IntegrityError):
        N.archive_validate(b"nope")
    assert b"truncated header" in lib.rinr_last_error()
    assert N.archive_validate(N.host_view(_tiny())) == 1
    assert lib.rinr_last_error() == b""


def _tiny():
    from paper_2306_16699_b200 import synth
    return synth.archive_bytes(synth.seeded_batch(synth.ARCH_A, [0]))


def test_threaded_validation_reports_first_failure():
    """Archives of >= 4096 records are checked on host threads; the error is
    still the first failing record in index order (archive.py:369-379)."""
    from paper_2306_16699_b200 import IntegrityError, synth
    mb = synth.tweak_r1(synth.random_batch(synth.ARCH_A, 10000, seed=4))
    data = bytearray(synth.archive_bytes(mb))
    assert N.archive_validate(bytes(data)) == 10000
    for k in (7000, 3000):  # flip one byte inside each record's body
        off, length = struct.unpack_from("<QI", data, 10 + 12 * k)
        data[off + length // 2] ^= 0xFF
    with pytest.raises(IntegrityError) as e:
        N.archive_validate(bytes(data))
    assert "record 3000" in str(e.value)
