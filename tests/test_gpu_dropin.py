"""The reference-facing drop-ins: decode / decode_batch on in-memory models
(decoder.py:19-61) through install() into a rinr-shaped package, and batches
that mix architectures, quantisation layouts, weight dtypes and source sizes
(grouped into one serialisation + one launch per group, order preserved)."""

import sys
import types
from dataclasses import dataclass

import numpy as np
import pytest

from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu


def _fake_rinr():
    """A minimal package with the reference's module layout (__init__.py:8-25):
    rinr.decoder.decode[_batch], rinr.image.ImageBuffer, rinr.bench.bench."""
    pkg = types.ModuleType("fakerinr")
    pkg.__path__ = []
    dec, img, bench = (types.ModuleType(f"fakerinr.{m}") for m in ("decoder", "image", "bench"))

    @dataclass
    class ImageBuffer:  # the reference's validating value type (image.py:12-30)
        pixels: np.ndarray

        def __post_init__(self):
            if self.pixels.min() < 0 or self.pixels.max() > 1:
                raise ValueError("range")

    img.ImageBuffer = ImageBuffer
    dec.decode = dec.decode_batch = pkg.decode = pkg.decode_batch = None
    bench.bench = None
    pkg.decoder, pkg.image, pkg.bench = dec, img, bench
    for m in (pkg, dec, img, bench):
        sys.modules[m.__name__] = m
    return pkg


def test_install_rebinds_fake_package():
    from paper_2306_16699_b200 import decoder, harness, synth
    pkg = _fake_rinr()
    try:
        decoder.install(pkg)
        assert pkg.decode_batch.__wrapped__ is decoder.decode_batch
        assert pkg.decoder.decode_batch.__wrapped__ is decoder.decode_batch
        assert pkg.decode.__wrapped__ is decoder.decode and pkg.decoder.decode.__wrapped__ is decoder.decode
        assert pkg.bench.bench is harness.bench
        models = [synth.config2(6, 0).model(i) for i in range(6)]
        imgs = pkg.decode_batch(models, 32, 32)
        assert all(type(im) is pkg.image.ImageBuffer for im in imgs)
        want = np.stack(O.decode_batch(O.read_models(synth.archive_bytes(synth.config2(6, 0))), 32, 32))
        got = np.stack([im.pixels for im in imgs])
        assert float(np.abs(got - want).max()) <= 1e-3
        one = pkg.decoder.decode(models[2], 7, 9)
        assert type(one) is pkg.image.ImageBuffer and one.pixels.shape == (7, 9, 3)
    finally:
        decoder._image_cls = decoder.ImageBuffer
        for name in [k for k in sys.modules if k == "fakerinr" or k.startswith("fakerinr.")]:
            del sys.modules[name]


def test_mixed_batch_groups_keep_order():
    from paper_2306_16699_b200 import compressor, decode_batch, synth
    from paper_2306_16699_b200.archive import ArchiveRecord, DatasetArchive, serialize
    a_q = [synth.config2(3, 0).model(i) for i in range(3)]            # [2,15,15,3] affine8, pruned
    a_f = [synth.config1(3).model(i) for i in range(3)]               # dense f32
    c_q = [synth.config3(2, 0).model(i) for i in range(2)]            # [2,40x9,3] affine8
    half = [compressor.to_half(synth.config1(2).model(i)) for i in range(2)]  # f16 weights
    for j, m in enumerate(a_f):
        m.source_h, m.source_w = 20 + j, 12
    models = [a_q[0], c_q[0], a_f[0], half[0], a_q[1], a_f[1], c_q[1], half[1], a_q[2], a_f[2]]
    imgs = decode_batch(models)  # source sizes differ per model
    data = serialize(DatasetArchive([ArchiveRecord(f"m{i}", m) for i, m in enumerate(models)]))
    ref = O.read_models(data)
    for i, (im, m) in enumerate(zip(imgs, ref)):
        want = O.decode(m)
        assert im.pixels.shape == want.shape, i
        assert float(np.abs(im.pixels - want).max()) <= 1e-3, i
