"""The vectorised producer (compressor + archive writer + synth) must emit
exactly the bytes the reference writer emits for the same models
(archive.py:92-184, compressor.py:109-218)."""

import numpy as np
import pytest

from oracle import rinr_oracle as O
from paper_2306_16699_b200 import archive, compressor, net, synth
from paper_2306_16699_b200.compressor import ModelBatch


def test_c1_bytes(golden):
    mb = synth.seeded_batch(synth.ARCH_A, range(8))
    assert synth.archive_bytes(mb) == golden("c1_r0")["archive"].tobytes()
    mb = synth.tweak_r1(synth.seeded_batch(synth.ARCH_A, range(16)))
    assert synth.archive_bytes(mb) == golden("c1_r1")["archive"].tobytes()


def test_c2_bytes(golden):
    assert synth.archive_bytes(synth.config2(32, 0)) == golden("c2")["archive"].tobytes()


def test_c3_bytes(golden):
    assert synth.archive_bytes(synth.config3(3, 0)) == golden("c3")["archive"].tobytes()


def test_zoo_roundtrip_bytes(golden):
    """Re-serialising the reference's own records (materialised by the
    oracle) through our writer gives the reference bytes back — covers f16,
    affine16, const layers, every form and mixed architectures."""
    data = golden("zoo")["archive"].tobytes()
    models = O.read_models(data)
    recs = []
    for i, om in enumerate(models):
        arch = net.Architecture(om.dims, om.omega)
        layers = [net.LayerWeights(l.w, l.b) for l in om.layers]
        quant = None
        if om.quant is not None:
            quant = compressor.QuantInfo(om.quant_mode, {k: compressor.LayerQuant(*v) for k, v in om.quant.items()})
        m = net.InrModel(arch, layers, [l.mask for l in om.layers], om.source_h, om.source_w, quant)
        recs.append(archive.ArchiveRecord(f"img{i:08d}", m))
    assert archive.serialize(archive.DatasetArchive(recs)) == data


def test_single_model_api_matches_batch():
    m = net.init(synth.ARCH_A, 3)
    m.source_h = m.source_w = 32
    p = compressor.quantize(compressor.prune_l1(m, 0.2), "affine8")
    mb = compressor.quantize_batch(compressor.prune_l1_batch(ModelBatch.from_models([m]), 0.2), "affine8")
    assert archive.encode_record(archive.ArchiveRecord("x", p)) == archive.encode_batch(mb, ["x"])[0]


def test_structural_and_format_errors():
    m = net.init(net.Architecture((2, 1, 3)), 0)
    with pytest.raises(Exception, match="entire layer"):
        compressor.prune_l1(m, 0.9)
    q = compressor.quantize(net.init(synth.ARCH_A, 0), "affine8")
    with pytest.raises(Exception, match="already quantized"):
        compressor.quantize(q, "affine8")


def test_large_store_is_valid():
    data = synth.large_store_bytes("c2", 3000, seed=1, chunk=1024)
    models = O.read_models(data)
    assert len(models) == 3000
    ratios = [1 - sum(l.mask.sum() for l in m.layers) / 300 for m in models]
    assert 0.10 < float(np.mean(ratios)) < 0.20  # PAPER.md:332 reports 15.6% for CIFAR-10
