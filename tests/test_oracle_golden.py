"""Pin the CPU oracle to the real reference: every golden vector produced by
running /root/reference (tests/golden/make_golden.py) must be reproduced
bit-for-bit by oracle/rinr_oracle.py."""

import numpy as np
import pytest

from conftest import STORE_CASES
from oracle import rinr_oracle as O


@pytest.mark.parametrize("case", STORE_CASES)
def test_materialize_bit_exact(golden, case):
    g = golden(case)
    models = O.read_models(g["archive"].tobytes())
    assert len(models) == g["params"].shape[0]
    for i, m in enumerate(models):
        f = O.flat_params(m)
        np.testing.assert_array_equal(f.view(np.uint32), g["params"][i, :f.size].view(np.uint32))


@pytest.mark.parametrize("case", STORE_CASES)
def test_decode_bit_exact(golden, case):
    g = golden(case)
    models = O.read_models(g["archive"].tobytes())
    for key in g:
        if not key.startswith("decode_"):
            continue
        h, w = map(int, key[len("decode_"):].split("x"))
        want = g[key]
        got = np.stack(O.decode_batch(models[:want.shape[0]], h, w))
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_grids(golden):
    g = golden("grids")
    for key, want in g.items():
        h, w = map(int, key[len("grid_"):].split("x"))
        np.testing.assert_array_equal(O.coordinate_grid(h, w), want)
        # the closed form the CUDA kernels use: f32(f64(i) * (1/(n-1))), last = 1
        for n, col in ((w, 0), (h, 1)):
            if n > 1:
                closed = (np.arange(n, dtype=np.float64) * (1.0 / (n - 1))).astype(np.float32)
                closed[-1] = 1.0
            else:
                closed = np.zeros(1, np.float32)
            axis = want[:, col].reshape(h, w)
            np.testing.assert_array_equal(axis[0, :] if col == 0 else axis[:, 0], closed)


def test_augment_checker_matches_reference_forward(golden):
    g = golden("augment")
    models = O.read_models(golden("c2")["archive"].tobytes())
    for key in g:
        if not key.startswith("raw_"):
            continue
        _, mode, i = key.split("_")
        mode, i = int(mode), int(i)
        coords, valid = O.augment_coords(32, 32, mode, g[f"params_{mode}_{i}"])
        np.testing.assert_array_equal(valid, g[f"valid_{mode}_{i}"])
        np.testing.assert_array_equal(O.forward(models[i], coords).view(np.uint32), g[key].view(np.uint32))


def test_known_answers(golden):
    k = golden("kat")
    assert list(k["param_count"]) == [9, 333, 13363]
    np.testing.assert_allclose(k["sin15_forward"], np.sin(np.float32(15.0)), rtol=0, atol=1e-6)
    m = O.OModel((2, 1, 3), 30.0, [O.OLayer(np.array([[1.0, 0.0]], np.float32), np.zeros(1, np.float32),
                                            np.ones((1, 2), bool)),
                                   O.OLayer(np.ones((3, 1), np.float32), np.zeros(3, np.float32),
                                            np.ones((3, 1), bool))])
    np.testing.assert_array_equal(O.forward(m, np.array([[0.5, 0.0]], np.float32)), k["sin15_forward"])


def test_u8_round_half_away():
    px = np.array([0.0, 1.0, 0.5 / 255, 1.5 / 255, 0.999, -0.1, 1.2], np.float32)
    assert list(O.to_u8(px)) == [0, 255, 1, 2, 255, 0, 255]


def test_integrity_errors(golden):
    data = bytearray(golden("c2")["archive"].tobytes())
    bad = bytearray(data)
    bad[-1] ^= 0xFF
    with pytest.raises(O.OracleIntegrityError, match="record 31: CRC mismatch"):
        O.read_models(bytes(bad))
    with pytest.raises(O.OracleIntegrityError, match="bad magic"):
        O.read_models(b"XXXX" + bytes(data[4:]))
    with pytest.raises(O.OracleIntegrityError, match="truncated"):
        O.read_models(bytes(data[:-10]))


# ---- encoder-side transforms (compressor.py:100-218, metrics.py:23-41) ---------

def test_transforms_oracle(golden):
    from transforms_common import case, cat
    g = golden("transforms")
    for name in g["names"]:
        name = str(name)
        dims, w, m, b = case(g, name)
        if f"{name}/ratio" in g:
            ratio, scope = float(g[f"{name}/ratio"]), str(g[f"{name}/scope"])
            if f"{name}/prune_error" in g:
                with pytest.raises(O.OracleStructuralError):
                    O.prune_l1(w, m, ratio, scope)
                continue
            w, m = O.prune_l1(w, m, ratio, scope)
            np.testing.assert_array_equal(cat(w).view(np.uint32), g[f"{name}/pw"])
            np.testing.assert_array_equal(cat(m).astype(np.uint8), g[f"{name}/pmask"])
        for mode, bits in (("affine8", 8), ("affine16", 16)):
            if f"{name}/{mode}/w" not in g:
                continue
            qw, info = O.quantize(w, m, b, bits)
            np.testing.assert_array_equal(cat(qw).view(np.uint32), g[f"{name}/{mode}/w"])
            lay = sorted(info)
            np.testing.assert_array_equal([info[i][2] for i in lay], g[f"{name}/{mode}/const"])
            if f"{name}/{mode}/scale" in g:
                np.testing.assert_array_equal(np.array([info[i][0] for i in lay]).view(np.uint64),
                                              g[f"{name}/{mode}/scale"].view(np.uint64))
                np.testing.assert_array_equal([info[i][1] for i in lay], g[f"{name}/{mode}/zp"])
            for i in lay:
                if not info[i][2]:
                    np.testing.assert_array_equal(O.quantize_codes(qw[i], info[i][0], info[i][1], bits).ravel(),
                                                  g[f"{name}/{mode}/codes{i}"])
    a, b2 = g["psnr/a"], g["psnr/b"]
    for k in range(a.shape[0]):
        assert O.psnr(a[k], b2[k]) == g["psnr/f"][k]
        assert O.psnr(a[k], b2[k], quantized=True) == g["psnr/q"][k]


# ---- training (net.py:152-300, encoder.py:28-85) --------------------------------

def test_training_oracle(golden):
    from transforms_common import split, split_bias
    g = golden("encoder")
    dims = (2, 15, 15, 3)
    coords = O.coordinate_grid(16, 16)
    imgs = g["images16"]
    for k in (0, 1):
        ws = split(g[f"grad{k}/w"], dims)
        bs = split_bias(g[f"grad{k}/b"], dims)
        ms = split(g[f"grad{k}/mask"], dims, bool)
        if k == 0:
            iw, ib, im = O.init_model(dims, int(g[f"grad{k}/seed"]))
            for a, b in zip(iw, ws):
                np.testing.assert_array_equal(a, b)
        loss, gws, gbs = O.loss_and_grad(ws, bs, ms, 30.0, coords, imgs[k].reshape(-1, 3))
        assert loss == g[f"grad{k}/loss"]
        np.testing.assert_array_equal(np.concatenate([x.ravel() for x in gws]), g[f"grad{k}/gw"])
        np.testing.assert_array_equal(np.concatenate([x.ravel() for x in gbs]), g[f"grad{k}/gb"])
    ws, bs, ms = O.init_model(dims, 33)
    curve = O.train(ws, bs, ms, 30.0, coords, imgs[2].reshape(-1, 3), 5e-4, 40)
    np.testing.assert_array_equal(curve, g["train/curve"])
    np.testing.assert_array_equal(np.concatenate([x.ravel() for x in ws]), g["train/w"])
    np.testing.assert_array_equal(np.concatenate([x.ravel() for x in bs]), g["train/b"])


def test_fitted_oracle(golden):
    """The oracle reproduces the reference decode of reference-fitted INRs
    bit for bit, and its PSNR against the source images (metrics.py:23-41)."""
    g = golden("fitted")
    for name in ("A", "C"):
        models = O.read_models(g[f"{name}/archive"].tobytes())
        got = np.stack(O.decode_batch(models))
        np.testing.assert_array_equal(got.view(np.uint32), g[f"{name}/decode"].view(np.uint32))
        for i in range(len(models)):
            assert abs(O.psnr(got[i], g[f"{name}/source"][i]) - g[f"{name}/psnr"][i]) <= 1e-9


def test_wide_training_oracle(golden):
    """The oracle's loss_and_grad / train on the wide and deep nets the
    general GPU encoder handles (reference fixtures: encoder.npz 'wgrad*',
    'wtrain')."""
    from transforms_common import split, split_bias
    g = golden("encoder")
    dims = (2, *[40] * 9, 3)
    coords = O.coordinate_grid(12, 12)
    for k in (0, 1):
        ws = split(g[f"wgrad{k}/w"], dims)
        bs = split_bias(g[f"wgrad{k}/b"], dims)
        ms = split(g[f"wgrad{k}/mask"], dims, bool)
        loss, gws, gbs = O.loss_and_grad(ws, bs, ms, 30.0, coords, g["images12"][k].reshape(-1, 3))
        assert abs(loss - g[f"wgrad{k}/loss"]) <= 1e-12 * g[f"wgrad{k}/loss"]
        np.testing.assert_allclose(np.concatenate([x.ravel() for x in gws]), g[f"wgrad{k}/gw"], rtol=1e-5, atol=1e-9)
    d4 = (2, 32, 32, 32, 3)
    ws, bs, ms = O.init_model(d4, 44)
    curve = O.train(ws, bs, ms, 30.0, coords, g["images12"][1].reshape(-1, 3), 2e-4, 20)
    np.testing.assert_allclose(curve, g["wtrain/curve"], rtol=1e-6)
