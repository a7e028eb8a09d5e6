"""GPU .rinr writer (csrc/writer.cu) vs the host writer, which is itself
byte-identical to the reference writer (tests/test_archive_writer.py,
archive.py:92-184): same models in -> same archive bytes out, for
unquantised f32 and affine8 / affine16 records, every layer form (dense,
dense + bitset, sparse), constant quantised layers and several
architectures."""

import numpy as np
import pytest
import torch

from paper_2306_16699_b200 import synth, transforms as T
from paper_2306_16699_b200.archive import serialize_batch
from paper_2306_16699_b200.net import Architecture

pytestmark = pytest.mark.gpu


def _batch(arch, n, seed):
    mb = synth.tweak_r1(synth.random_batch(arch, n, seed))
    rng = np.random.default_rng(seed)
    for b in mb.b:
        b[:] = rng.normal(0, 0.05, b.shape).astype(np.float32)
    if len(arch.dims) > 3:  # a constant hidden layer in record 1 (quantize -> constant)
        mb.w[1][1] = np.float32(0.01)
    return mb


@pytest.mark.parametrize("dims", [(2, 15, 15, 3), (2, *[40] * 9, 3), (2, 8, 8, 8, 3), (2, 5, 3)])
@pytest.mark.parametrize("mode", [None, "affine8", "affine16"])
def test_gpu_writer_bytes(dims, mode):
    arch = Architecture(dims)
    n = 12
    mb = _batch(arch, n, seed=len(dims) * 7 + (0 if mode is None else 3))
    mb.source_h, mb.source_w = 32, 24
    dm = T.DeviceModels.from_batch(mb)
    # per-record ratios: dense (0), dense + bitset (~5%), sparse (20-50%)
    ratios = torch.tensor([0.0, 0.05, 0.2, 0.5] * (n // 4), dtype=torch.float64)
    T.prune_l1(dm, ratios, check=False)
    q = T.quantize(dm, mode) if mode is not None and len(dims) > 3 else None
    got = T.serialize(dm, q, id_prefix="img", first_id=5, id_width=8).cpu().numpy().tobytes()
    host = T.quantized_batch(dm, q) if q is not None else dm.to_batch()
    want = serialize_batch(host, [f"img{5 + i:08d}" for i in range(n)])
    assert got == want


def test_gpu_writer_ids_and_store_roundtrip():
    from oracle import rinr_oracle as O
    from paper_2306_16699_b200 import Store
    mb = synth.config2(40, seed=3)
    dm = T.DeviceModels.from_batch(mb)
    got = T.serialize(dm, None, id_prefix="rec-", first_id=99_999_998, id_width=3).cpu().numpy().tobytes()
    want = serialize_batch(dm.to_batch(), [f"rec-{99_999_998 + i:03d}" for i in range(40)])
    assert got == want
    with Store(got) as st:
        assert st.record_meta(39)["id"] == "rec-100000037"
        params = st.dequantize(torch.arange(40)).cpu().numpy()
    for i, m in enumerate(O.read_models(got)):
        f = O.flat_params(m)
        np.testing.assert_array_equal(params[i, :f.size].view(np.uint32), f.view(np.uint32))
