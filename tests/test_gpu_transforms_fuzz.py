"""Randomised parity sweep of GPU prune_l1 + quantize (csrc/transforms.cu)
against the oracle (compressor.py:108-218 restated): random architectures on
every kernel path (register-resident keys for global scope with P <= 512,
warp per model for P <= 2048, CTA per model above), random batch sizes, per-model ratios in [0, 0.99), both scopes, existing masks,
8 and 16 bits, and adversarial weights (magnitude ties, signed zeros,
denormals, constant and single-survivor layers).

Bar: bit-exact weights / masks / scales / zero points / codes; per-model
status equal to the oracle's outcome (StructuralError / NumericError), with
failing models left unchanged."""

import os

import numpy as np
import pytest
import torch

from oracle import rinr_oracle as O
from transforms_common import cat, split

pytestmark = pytest.mark.gpu

ARCHS = [(2, 15, 15, 3), (2, 16, 16, 3), (2, 7, 9, 3), (2, 8, 8, 8, 3), (2, 32, 32, 32, 32, 3),
         (2, 40, 40, 40, 3), (2, 64, 64, 64, 3), (2, 24, 12, 3), (2, 3), (2, 5, 3), (2, 20, 20, 3),
         (2, 11, 11, 11, 3)]


def _model(rng, dims):
    w = [rng.normal(0, 0.3 if l == 0 else 0.05, (dims[l + 1], dims[l])).astype(np.float32)
         for l in range(len(dims) - 1)]
    kind = rng.integers(6)
    if kind == 0:  # coarse grid: many exact magnitude ties, signed zeros
        w = [(np.round(x * 16) / 16).astype(np.float32) for x in w]
        w[-1].flat[0] = np.float32(-0.0)
    elif kind == 1:  # denormals and tiny values
        for x in w:
            x.flat[::7] = np.float32(1e-40) * rng.choice([-1, 1], x.flat[::7].shape)
    elif kind == 2 and len(w) > 2:  # a constant hidden layer
        w[1][:] = np.float32(rng.normal(0, 0.1))
    elif kind == 3:  # all weights equal magnitude
        w = [np.where(rng.random(x.shape) < 0.5, -0.25, 0.25).astype(np.float32) for x in w]
    m = [np.ones(x.shape, bool) for x in w]
    if rng.random() < 0.4:  # already pruned: masked entries are zero
        for i in range(len(w)):
            m[i] = rng.random(w[i].shape) >= rng.uniform(0, 0.5)
            if not m[i].any():
                m[i].flat[0] = True
            w[i] = np.multiply(w[i], m[i])
    if kind == 4 and len(w) > 2:  # a single surviving hidden weight
        m[1][:] = False
        m[1].flat[int(rng.integers(m[1].size))] = True
        w[1] = np.multiply(w[1], m[1])
    b = [rng.normal(0, 0.1, dims[l + 1]).astype(np.float32) for l in range(len(dims) - 1)]
    return w, m, b


@pytest.mark.parametrize("seed", range(int(os.environ.get("RINR_FUZZ_SEEDS", 32))))
def test_transforms_fuzz(seed):
    from paper_2306_16699_b200 import transforms as T
    from paper_2306_16699_b200.net import Architecture
    rng = np.random.default_rng(5000 + seed)
    dims = ARCHS[int(rng.integers(len(ARCHS)))]
    n = int(rng.integers(1, 48))
    models = [_model(rng, dims) for _ in range(n)]
    ratios = rng.choice([0.0, 0.1, 0.5, 0.9, 0.99], n) * rng.random(n) ** 0.3
    if rng.random() < 0.2:
        ratios[int(rng.integers(n))] = 0.999  # likely zeroes a layer -> StructuralError
    scope = str(rng.choice(["global", "per_layer"]))
    bits = int(rng.choice([8, 16]))
    dm = T.DeviceModels(Architecture(dims),
                        torch.from_numpy(np.stack([cat(w) for w, _, _ in models]).astype(np.float32)).cuda(),
                        torch.from_numpy(np.stack([cat(m) for _, m, _ in models]).astype(np.uint8)).cuda(),
                        torch.from_numpy(np.stack([cat(b) for _, _, b in models]).astype(np.float32)).cuda())
    w_in, m_in = dm.w.cpu().numpy().copy(), dm.mask.cpu().numpy().copy()
    st = T.prune_l1(dm, torch.from_numpy(ratios), scope, check=False).cpu().numpy()
    w_p, m_p = dm.w.cpu().numpy().copy(), dm.mask.cpu().numpy().copy()
    pruned = []
    for k, (w, m, b) in enumerate(models):
        try:
            pw, pm = O.prune_l1(w, m, float(ratios[k]), scope)
        except O.OracleStructuralError:
            assert st[k] != 0, (seed, k)
            np.testing.assert_array_equal(w_p[k].view(np.uint32), w_in[k].view(np.uint32))
            np.testing.assert_array_equal(m_p[k], m_in[k])
            pruned.append((w, m, b))
            continue
        assert st[k] == 0, (seed, k, st[k])
        np.testing.assert_array_equal(m_p[k], cat(pm).astype(np.uint8), err_msg=f"seed {seed} model {k}")
        np.testing.assert_array_equal(w_p[k].view(np.uint32), cat(pw).view(np.uint32), err_msg=f"seed {seed} model {k}")
        pruned.append((pw, pm, b))
    q = T.quantize(dm, "affine8" if bits == 8 else "affine16", check=False)
    assert not q.status.any()
    w_q = dm.w.cpu().numpy()
    codes = q.codes.cpu().numpy().view(np.uint16)
    for k, (w, m, b) in enumerate(pruned):
        qw, info = O.quantize(w, m, b, bits)
        np.testing.assert_array_equal(w_q[k].view(np.uint32), cat(qw).view(np.uint32), err_msg=f"seed {seed} model {k}")
        for i, (scale, zp, const) in info.items():
            assert bool(q.constant[k, i - 1]) == const, (seed, k, i)
            assert q.scale[k, i - 1].item() == scale and q.zero_point[k, i - 1].item() == zp, (seed, k, i)
            if not const:
                np.testing.assert_array_equal(split(codes[k], dims)[i], O.quantize_codes(qw[i], scale, zp, bits))


@pytest.mark.gpu
@pytest.mark.parametrize("bits,arch", [(8, (2, 15, 15, 3)), (16, (2, 15, 15, 3)), (8, (2, 40, 40, 40, 40, 40, 40, 40, 40, 40, 3))])
def test_quantize_half_step_weights(bits, arch):
    """Weights on and one float ulp either side of mn + (k + 1/2) scale: the
    f64 quotient w / scale lands next to a rounding boundary, so the GPU's
    reciprocal + FMA quotient must round exactly like the oracle's true
    division (compressor.py:180-202 via O.quantize)."""
    from paper_2306_16699_b200 import transforms as T
    from paper_2306_16699_b200.net import Architecture
    rng = np.random.default_rng(77 + bits)
    qmax = (1 << bits) - 1
    models = []
    for _ in range(24):
        w, m, b = _model(rng, arch)
        m = [np.ones_like(x, dtype=bool) for x in m]
        for i in range(1, len(arch) - 2):
            lo, hi = np.float32(rng.uniform(-2, -0.01)), np.float32(rng.uniform(0.01, 2))
            scale = (float(hi) - float(lo)) / qmax
            k = rng.integers(0, qmax, w[i].size)
            v = (float(lo) + (k + 0.5) * scale).astype(np.float32)
            v = np.where(rng.random(v.size) < 1 / 3, np.nextafter(v, np.float32(-9)),
                         np.where(rng.random(v.size) < 0.5, np.nextafter(v, np.float32(9)), v))
            v[0], v[1] = lo, hi
            w[i] = v.reshape(w[i].shape).astype(np.float32)
        models.append((w, m, b))
    dm = T.DeviceModels(Architecture(arch),
                        torch.from_numpy(np.stack([cat(w) for w, _, _ in models]).astype(np.float32)).cuda(),
                        torch.from_numpy(np.stack([cat(m) for _, m, _ in models]).astype(np.uint8)).cuda(),
                        torch.from_numpy(np.stack([cat(b) for _, _, b in models]).astype(np.float32)).cuda())
    q = T.quantize(dm, "affine8" if bits == 8 else "affine16", check=False)
    assert not q.status.any()
    w_q = dm.w.cpu().numpy()
    codes = q.codes.cpu().numpy().view(np.uint16)
    for k, (w, m, b) in enumerate(models):
        qw, info = O.quantize(w, m, b, bits)
        np.testing.assert_array_equal(w_q[k].view(np.uint32), cat(qw).view(np.uint32), err_msg=f"model {k}")
        for i, (scale, zp, const) in info.items():
            if not const:
                np.testing.assert_array_equal(split(codes[k], arch)[i], O.quantize_codes(qw[i], scale, zp, bits))
