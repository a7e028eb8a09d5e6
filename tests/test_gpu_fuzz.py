"""Randomised parity sweep of the decode path against the oracle: random
architectures (uniform narrow / wide, ragged), prune ratios, quantisation
modes (none / affine8 / affine16 / f16 weights), record forms, mixed-arch
stores, output sizes, precisions, layouts, dtypes and augment modes.  Every
case builds an archive with the writer, decodes through the C ABI and checks
the stated bars (fp32 / exact: max-abs <= 1e-3 in [0,1]; bf16: PSNR >= conftest.bf16_bar;
dequantised weights bit-exact)."""

import os

import numpy as np
import pytest
import torch

from conftest import bf16_bar
from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu

ARCHS = [(2, 15, 15, 3), (2, 16, 16, 3), (2, 8, 8, 8, 3), (2, 32, *[32] * 8, 3), (2, *[40] * 9, 3),
         (2, 7, 11, 3), (2, 3), (2, 24, 12, 3)]


def _random_store(rng):
    from paper_2306_16699_b200 import compressor, synth
    from paper_2306_16699_b200.archive import ArchiveRecord, DatasetArchive, serialize
    from paper_2306_16699_b200.net import Architecture
    mixed = rng.random() < 0.3
    records = []
    for part in range(2 if mixed else 1):
        dims = ARCHS[int(rng.integers(len(ARCHS)))]
        n = int(rng.integers(1, 6))
        mb = synth.tweak_r1(synth.seeded_batch(Architecture(dims, float(rng.choice([30.0, 20.0]))),
                                               [int(x) for x in rng.integers(0, 10 ** 6, n)],
                                               (int(rng.integers(4, 40)), int(rng.integers(4, 40)))))
        for b in mb.b:
            b[:] = rng.normal(0, 0.05, b.shape).astype(np.float32)
        ratio = float(rng.choice([0.0, 0.05, 0.2, 0.45]))
        if ratio > 0:
            mb = compressor.prune_l1_batch(mb, ratio)
        mode = rng.choice(["none", "affine8", "affine16", "f16"])
        if mode in ("affine8", "affine16") and len(dims) > 3:
            mb = compressor.quantize_batch(mb, str(mode))
        models = [mb.model(i) for i in range(mb.n)]
        if mode == "f16":
            models = [compressor.to_half(m) for m in models]
        records += models
    arc = DatasetArchive([ArchiveRecord(f"r{i}", m) for i, m in enumerate(records)])
    return serialize(arc)


@pytest.mark.parametrize("seed", range(int(os.environ.get("RINR_FUZZ_SEEDS", 40))))
def test_decode_fuzz(seed):
    from paper_2306_16699_b200 import Store
    rng = np.random.default_rng(1000 + seed)
    data = _random_store(rng)
    models = O.read_models(data)
    n = len(models)
    with Store(data) as st:
        # dequant bit-exact
        got = st.dequantize(torch.arange(n)).cpu().numpy()
        for i, m in enumerate(models):
            want = O.flat_params(m)
            np.testing.assert_array_equal(got[i, :want.size].view(np.uint32), want.view(np.uint32))
        for _ in range(3):
            h, w = int(rng.integers(1, 70)), int(rng.integers(1, 70))
            precision = str(rng.choice(["exact", "fp32", "bf16"]))
            sin = str(rng.choice(["mufu", "accurate"]))
            ids = torch.from_numpy(rng.integers(0, n, int(rng.integers(1, 9))).astype(np.int64))
            aug_mode = rng.choice([None, "offset", "crop"])
            kw = {}
            if aug_mode is not None:
                if aug_mode == "offset":
                    aug = torch.tensor([[float(rng.integers(0, 9)), float(rng.integers(0, 9)),
                                         float(rng.integers(0, 2)), 4.0, 0.0] for _ in range(len(ids))])
                else:
                    sx, sy = rng.uniform(0.3, 1.0, 2)
                    aug = torch.tensor([[float(rng.uniform(0, 1 - sx)), float(rng.uniform(0, 1 - sy)), float(sx),
                                         float(sy), float(rng.integers(0, 2))] for _ in range(len(ids))])
                kw = dict(aug=aug, aug_mode=str(aug_mode))
            out = st.decode(ids, h, w, layout="nhwc", precision=precision, sin=sin, **kw).cpu().numpy()
            for j, k in enumerate(ids.tolist()):
                if aug_mode is None:
                    want = O.decode(models[k], h, w)
                else:
                    mode = O.AUG_OFFSET if aug_mode == "offset" else O.AUG_CROP
                    want = O.decode_augmented(models[k], h, w, mode, aug[j].numpy(), (0, 0, 0), (1, 1, 1))
                    want = want.transpose(1, 2, 0)
                if precision == "bf16":
                    assert O.psnr(out[j], want) >= bf16_bar(models[k].dims), (seed, precision, h, w, aug_mode)
                else:
                    assert float(np.abs(out[j] - want).max()) <= 1e-3, (seed, precision, sin, h, w, aug_mode)
