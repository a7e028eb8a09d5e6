"""SPEC known answers through the GPU decode (SPEC.md line
numbers below are the reference's).  Each builds records with the writer
and decodes them with the fused kernels via the C ABI."""

import numpy as np
import pytest
import torch

from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu
PRECISIONS = ["exact", "fp32", "bf16"]


def _store_bytes(models):
    from paper_2306_16699_b200 import ArchiveRecord, DatasetArchive, serialize
    return serialize(DatasetArchive([ArchiveRecord(f"m{i}", m) for i, m in enumerate(models)]))


def _model(dims, ws, bs, h=4, w=4, omega=30.0):
    from paper_2306_16699_b200 import Architecture, InrModel, LayerWeights
    layers = [LayerWeights(np.asarray(a, np.float32), np.asarray(b, np.float32)) for a, b in zip(ws, bs)]
    masks = [np.ones(l.w.shape, bool) for l in layers]
    return InrModel(Architecture(tuple(dims), omega), layers, masks, h, w)


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("dims", [(2, 15, 15, 3), (2, 40, 40, 40, 3), (2, 5, 3)])
def test_all_zero_model_is_black(precision, dims):
    """all-zero weights and biases give output (0, 0, 0)."""
    from paper_2306_16699_b200 import Store
    ws = [np.zeros((o, i)) for i, o in zip(dims[:-1], dims[1:])]
    bs = [np.zeros(o) for o in dims[1:]]
    with Store(_store_bytes([_model(dims, ws, bs)] * 3)) as st:
        out = st.decode(torch.arange(3), 24, 40, precision=precision).cpu()
    assert torch.count_nonzero(out) == 0


@pytest.mark.parametrize("sin", ["accurate", "mufu"])
def test_single_unit_sin15(sin):
    """one hidden unit w=[[1,0]], b=0, omega=30 at input (0.5, 0)
    gives sin(15) = 0.65028787 (the last layer routes it to R)."""
    from paper_2306_16699_b200 import Store
    dims = (2, 1, 3)
    m = _model(dims, [[[1.0, 0.0]], [[1.0], [0.0], [0.0]]], [[0.0], [0.0, 0.0, 0.0]], h=1, w=3)
    with Store(_store_bytes([m])) as st:
        out = st.decode(torch.arange(1), 1, 3, layout="nhwc", precision="exact", sin=sin).cpu().numpy()
    # pixel (row 0, col 1) is (x, y) = (0.5, 0)
    tol = 0.0 if sin == "accurate" else 2e-6
    assert abs(float(out[0, 0, 1, 0]) - 0.65028787) <= tol + 1e-8
    assert out[0, 0, 1, 1] == 0.0 and out[0, 0, 1, 2] == 0.0


@pytest.mark.parametrize("precision", ["exact", "fp32"])
def test_last_layer_linear(precision):
    """the last layer is exactly affine (no activation): halving
    its weights and bias halves the (unclamped) output."""
    from paper_2306_16699_b200 import Store, synth
    mb = synth.seeded_batch(synth.ARCH_A, range(4))
    for b in mb.b[-1]:
        b[:] = 0.25
    full = [mb.model(i) for i in range(4)]
    half = [mb.model(i) for i in range(4)]
    for m in half:
        m.layers[-1].w = (m.layers[-1].w * np.float32(0.5)).astype(np.float32)
        m.layers[-1].b = (m.layers[-1].b * np.float32(0.5)).astype(np.float32)
    with Store(_store_bytes(full)) as a, Store(_store_bytes(half)) as b:
        fa = a.decode(torch.arange(4), 16, 16, precision=precision).cpu().numpy()
        fb = b.decode(torch.arange(4), 16, 16, precision=precision).cpu().numpy()
    inside = (fa > 0.0) & (fa < 1.0)  # the clamp is the only non-linearity after the last layer
    assert inside.mean() > 0.5
    np.testing.assert_allclose(fb[inside], 0.5 * fa[inside], atol=2e-6)
    # and against the oracle
    want = np.stack(O.decode_batch(O.read_models(_store_bytes(full)), 16, 16)).transpose(0, 3, 1, 2)
    assert float(np.abs(fa - want).max()) <= 1e-3


@pytest.mark.parametrize("arch_name,precision", [("ARCH_A", "fp32"), ("ARCH_C", "bf16"), ("ARCH_C", "fp32"),
                                                 ("ZOO", "exact")])
def test_large_output_sampled(arch_name, precision):
    """Maximum-size path: 2048 x 2048 decodes on every kernel family, checked
    against the oracle's forward on sampled pixels (rows/cols at the edges
    and the middle)."""
    from paper_2306_16699_b200 import Store, synth
    if arch_name == "ZOO":
        mb = synth.tweak_r1(synth.seeded_batch(synth.Architecture((2, 7, 11, 3)), range(2)))
    else:
        mb = synth.tweak_r1(synth.seeded_batch(getattr(synth, arch_name), range(2)))
    data = synth.archive_bytes(mb)
    models = O.read_models(data)
    H = W = 2048
    with Store(data) as st:
        out = st.decode(torch.arange(2), H, W, layout="nhwc", precision=precision).cpu().numpy()
    assert np.isfinite(out).all() and out.min() >= 0.0 and out.max() <= 1.0
    xs = O.axis_coords(W)
    rows = [0, 1, 1023, 2046, 2047]
    cols = np.array([0, 1, 777, 1024, 2046, 2047])
    for i, m in enumerate(models):
        for r in rows:
            c = np.stack([xs[cols], np.full(len(cols), O.axis_coords(H)[r], np.float32)], 1)
            want = np.clip(O.forward(m, c), 0.0, 1.0)
            got = out[i, r, cols]
            if precision == "bf16":
                assert float(np.abs(got - want).max()) <= 2e-2
            else:
                assert float(np.abs(got - want).max()) <= 1e-3


def test_bench_harness(golden, tmp_path):
    """rinr.bench.bench mirror: report fields, stage keys, deterministic digest
    that matches a digest of the same u8 pixels computed independently."""
    import hashlib
    from paper_2306_16699_b200 import Store, bench
    data = golden("zoo")["archive"].tobytes()  # mixed architectures and native sizes
    p = tmp_path / "zoo.rinr"
    p.write_bytes(data)
    r1 = bench(str(p), batch=3)
    r2 = bench(data, batch=5, jobs=4)
    models = O.read_models(data)
    assert r1.images == len(models) and r1.pixels == sum(m.source_h * m.source_w for m in models)
    assert set(r1.stage_seconds) == {"load", "dequantize", "forward", "clamp_convert"}
    assert r1.digest == r2.digest and r1.images_per_s > 0
    h = hashlib.sha256()
    with Store(data) as st:
        for k, m in enumerate(models):
            u8 = st.decode(torch.tensor([k]), m.source_h, m.source_w, dtype=torch.uint8, layout="nhwc",
                           precision="exact", sin="accurate").cpu().numpy()[0]
            want = O.to_u8(O.decode(m))
            assert np.abs(u8.astype(int) - want.astype(int)).max() <= 1
            h.update(u8.tobytes())
    assert h.hexdigest() == r1.digest
