"""GPU parity of the encoder-side transforms (csrc/transforms.cu via the C ABI)
against the reference's outputs (tests/golden/transforms.npz, produced by
rinr.compressor / rinr.metrics) and against the oracle on larger random
batches.

Tolerances: prune masks, pruned / quantised weights (uint32), scales
(uint64), zero points and codes are bit-exact; PSNR is f64 with a different
summation order: relative difference <= 1e-12."""

import numpy as np
import pytest
import torch

from oracle import rinr_oracle as O
from transforms_common import case, cat, split, split_bias

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2306_16699_b200 import transforms
    return transforms


def _device_models(T, dims, ws, ms, bs):
    """Stack same-architecture models (lists of per-matrix arrays) on the GPU."""
    from paper_2306_16699_b200.net import Architecture
    w = torch.from_numpy(np.stack([cat(x) for x in ws]).astype(np.float32)).cuda()
    m = torch.from_numpy(np.stack([cat(x) for x in ms]).astype(np.uint8)).cuda()
    b = torch.from_numpy(np.stack([cat(x) for x in bs]).astype(np.float32)).cuda()
    return T.DeviceModels(Architecture(tuple(int(d) for d in dims)), w, m, b)


def test_prune_quantize_golden(golden, T):
    from paper_2306_16699_b200 import BatchItemError, StructuralError
    g = golden("transforms")
    for name in g["names"]:
        name = str(name)
        dims, w, m, b = case(g, name)
        dm = _device_models(T, dims, [w], [m], [b])
        if f"{name}/ratio" in g:
            ratio, scope = float(g[f"{name}/ratio"]), str(g[f"{name}/scope"])
            if f"{name}/prune_error" in g:
                w0 = dm.w.clone()
                with pytest.raises(BatchItemError) as e:
                    T.prune_l1(dm, ratio, scope)
                assert e.value.index == 0 and isinstance(e.value.cause, StructuralError)
                assert torch.equal(dm.w, w0)  # left unchanged
                continue
            T.prune_l1(dm, ratio, scope)
            np.testing.assert_array_equal(dm.w[0].cpu().numpy().view(np.uint32), g[f"{name}/pw"], err_msg=name)
            np.testing.assert_array_equal(dm.mask[0].cpu().numpy(), g[f"{name}/pmask"], err_msg=name)
        for mode in ("affine8", "affine16"):
            if f"{name}/{mode}/w" not in g:
                continue
            dq = T.DeviceModels(dm.arch, dm.w.clone(), dm.mask.clone(), dm.b.clone())
            q = T.quantize(dq, mode)
            np.testing.assert_array_equal(dq.w[0].cpu().numpy().view(np.uint32), g[f"{name}/{mode}/w"],
                                          err_msg=f"{name} {mode}")
            np.testing.assert_array_equal(q.constant[0].cpu().numpy(), g[f"{name}/{mode}/const"])
            if f"{name}/{mode}/scale" in g:
                np.testing.assert_array_equal(q.scale[0].cpu().numpy().view(np.uint64),
                                              g[f"{name}/{mode}/scale"].view(np.uint64))
                np.testing.assert_array_equal(q.zero_point[0].cpu().numpy(), g[f"{name}/{mode}/zp"])
            codes = q.codes[0].cpu().numpy().view(np.uint16)
            for i in range(1, len(dims) - 2):
                key = f"{name}/{mode}/codes{i}"
                if key in g:
                    np.testing.assert_array_equal(split(codes, dims)[i].ravel(), g[key], err_msg=key)


def _random_models(dims, n, seed):
    rng = np.random.default_rng(seed)
    ws, ms, bs = [], [], []
    for k in range(n):
        w = [rng.normal(0, 0.3 if l == 0 else 0.05, (dims[l + 1], dims[l])).astype(np.float32)
             for l in range(len(dims) - 1)]
        if k % 3 == 0:  # many magnitude ties and signed zeros
            w = [(np.round(x * 32) / 32).astype(np.float32) for x in w]
            w[1][0, :3] = np.float32(-0.0)
        ws.append(w)
        ms.append([np.ones(x.shape, bool) for x in w])
        bs.append([rng.normal(0, 0.1, dims[l + 1]).astype(np.float32) for l in range(len(dims) - 1)])
    return ws, ms, bs


@pytest.mark.parametrize("dims", [(2, 15, 15, 3), (2, 40, 40, 40, 3), (2, 7, 9, 3)])
def test_random_batches_vs_oracle(T, dims):
    n = 64
    ws, ms, bs = _random_models(dims, n, seed=sum(dims))
    ratios = np.random.default_rng(1).uniform(0.0, 0.7, n)
    dm = _device_models(T, dims, ws, ms, bs)
    T.prune_l1(dm, torch.from_numpy(ratios))
    q = T.quantize(dm, "affine8")
    w_gpu, m_gpu = dm.w.cpu().numpy(), dm.mask.cpu().numpy()
    codes = q.codes.cpu().numpy().view(np.uint16)
    for k in range(n):
        pw, pm = O.prune_l1(ws[k], ms[k], float(ratios[k]))
        np.testing.assert_array_equal(m_gpu[k], cat(pm).astype(np.uint8))
        qw, info = O.quantize(pw, pm, bs[k], 8)
        np.testing.assert_array_equal(w_gpu[k].view(np.uint32), cat(qw).view(np.uint32))
        for i, (scale, zp, const) in info.items():
            assert q.scale[k, i - 1].item() == scale and q.zero_point[k, i - 1].item() == zp
            assert bool(q.constant[k, i - 1]) == const
            if not const:
                np.testing.assert_array_equal(split(codes[k], dims)[i], O.quantize_codes(qw[i], scale, zp, 8))


def test_errors(T):
    from paper_2306_16699_b200 import BatchItemError, InvalidInputError, NumericError
    dims = (2, 15, 15, 3)
    ws, ms, bs = _random_models(dims, 4, seed=9)
    dm = _device_models(T, dims, ws, ms, bs)
    with pytest.raises(BatchItemError) as e:
        T.prune_l1(dm, torch.tensor([0.1, 0.2, 1.0, 0.3], dtype=torch.float64))
    assert e.value.index == 2 and isinstance(e.value.cause, InvalidInputError)
    dm.b[1, 5] = float("nan")
    w_before = dm.w.clone()
    with pytest.raises(BatchItemError) as e:
        T.quantize(dm, "affine8")
    assert e.value.index == 1 and isinstance(e.value.cause, NumericError)
    assert torch.equal(dm.w[1], w_before[1])  # model 1 untouched
    with pytest.raises(InvalidInputError):
        T.quantize(dm, "int4")


def test_psnr_golden(golden, T):
    g = golden("transforms")
    a, b = torch.from_numpy(g["psnr/a"]).cuda(), torch.from_numpy(g["psnr/b"]).cuda()
    for quantized, key in ((False, "psnr/f"), (True, "psnr/q")):
        _, p = T.psnr(a, b, quantized)
        p = p.cpu().numpy()
        want = g[key]
        assert np.isinf(p[3]) and np.isinf(want[3])
        np.testing.assert_allclose(p[:3], want[:3], rtol=1e-12, atol=0)


def test_roundtrip_to_archive(T):
    """GPU prune + quantize -> host ModelBatch -> writer -> store -> decode works
    and matches the oracle decode of the written archive."""
    from paper_2306_16699_b200 import Store, synth
    from paper_2306_16699_b200.compressor import ModelBatch
    mb = synth.tweak_r1(synth.seeded_batch(synth.ARCH_A, range(16)))
    dm = T.DeviceModels.from_batch(mb)
    T.prune_l1(dm, 0.2)
    q = T.quantize(dm, "affine8")
    out = T.quantized_batch(dm, q)
    assert isinstance(out, ModelBatch)
    data = synth.archive_bytes(out)
    models = O.read_models(data)
    with Store(data) as st:
        got = st.decode(torch.arange(16), 32, 32, layout="nhwc").cpu().numpy()
    want = np.stack(O.decode_batch(models, 32, 32))
    assert float(np.abs(got - want).max()) <= 1e-3
