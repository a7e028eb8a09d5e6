"""Host (numpy) producer transforms vs the reference's golden outputs
(tests/golden/transforms.npz, made by tests/golden/make_golden.py from
rinr.compressor): prune_l1 in both scopes (compressor.py:108-152) and
quantize (compressor.py:160-202), bit-exact."""

import numpy as np
import pytest

from paper_2306_16699_b200 import compressor
from paper_2306_16699_b200.compressor import ModelBatch
from paper_2306_16699_b200.errors import InvalidInputError, StructuralError
from paper_2306_16699_b200.net import Architecture
from transforms_common import case, cat


def _batch(dims, w, m, b):
    arch = Architecture(tuple(int(d) for d in dims))
    return ModelBatch(arch, [x[None].copy() for x in w], [x[None].astype(np.float32) for x in b],
                      [x[None].copy() for x in m])


def test_prune_quantize_golden(golden):
    g = golden("transforms")
    scopes = set()
    for name in g["names"]:
        name = str(name)
        dims, w, m, b = case(g, name)
        mb = _batch(dims, w, m, b)
        if f"{name}/ratio" in g:
            ratio, scope = float(g[f"{name}/ratio"]), str(g[f"{name}/scope"])
            scopes.add(scope)
            if f"{name}/prune_error" in g:
                with pytest.raises(StructuralError):
                    compressor.prune_l1_batch(mb, ratio, scope)
                continue
            mb = compressor.prune_l1_batch(mb, ratio, scope)
            np.testing.assert_array_equal(cat([x[0] for x in mb.w]).view(np.uint32), g[f"{name}/pw"])
            np.testing.assert_array_equal(cat([x[0] for x in mb.mask]).astype(np.uint8), g[f"{name}/pmask"])
            # the single-model wrapper agrees with the batch form
            one = compressor.prune_l1(_batch(dims, w, m, b).model(0), ratio, scope)
            np.testing.assert_array_equal(cat([l.w for l in one.layers]).view(np.uint32), g[f"{name}/pw"])
        for mode in ("affine8", "affine16"):
            if f"{name}/{mode}/w" not in g:
                continue
            q = compressor.quantize_batch(mb, mode)
            np.testing.assert_array_equal(cat([x[0] for x in q.w]).view(np.uint32), g[f"{name}/{mode}/w"])
            lay = sorted(q.quant)
            np.testing.assert_array_equal([bool(q.quant[i].constant[0]) for i in lay], g[f"{name}/{mode}/const"])
            if f"{name}/{mode}/scale" in g:
                np.testing.assert_array_equal(np.array([q.quant[i].scale[0] for i in lay]).view(np.uint64),
                                              g[f"{name}/{mode}/scale"].view(np.uint64))
                np.testing.assert_array_equal([int(q.quant[i].zero_point[0]) for i in lay], g[f"{name}/{mode}/zp"])
    assert scopes == {"global", "per_layer"}


def test_prune_scope_errors():
    arch = Architecture((2, 4, 3))
    rng = np.random.default_rng(0)
    w = [rng.standard_normal((1, 4, 2)).astype(np.float32), rng.standard_normal((1, 3, 4)).astype(np.float32)]
    mb = ModelBatch(arch, w, [np.zeros((1, 4), np.float32), np.zeros((1, 3), np.float32)],
                    [np.ones((1, 4, 2), bool), np.ones((1, 3, 4), bool)])
    with pytest.raises(InvalidInputError, match="unknown scope"):
        compressor.prune_l1_batch(mb, 0.1, "rows")
    with pytest.raises(InvalidInputError):
        compressor.prune_l1(mb.model(0), 1.0)
    # per-layer: each matrix keeps ceil((1 - r) * size) entries
    p = compressor.prune_l1_batch(mb, 0.5, "per_layer")
    assert [int(x.sum()) for x in p.mask] == [4, 6]


def test_cifar_ratios_vectorised():
    """synth.cifar_ratios == dynamic_ratio(cifar, psnr) per record (compressor.py:50-65)."""
    from paper_2306_16699_b200 import synth
    from paper_2306_16699_b200.compressor import dynamic_ratio_cifar
    rng = np.random.default_rng(11 + 7919)
    want = np.array([dynamic_ratio_cifar(p) for p in rng.uniform(28.0, 37.0, 5000)])
    np.testing.assert_array_equal(synth.cifar_ratios(5000, 11).view(np.uint64), want.view(np.uint64))
