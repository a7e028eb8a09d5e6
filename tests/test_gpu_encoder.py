"""GPU encoder (csrc/fit.cu) against the reference's own training results
(tests/golden/encoder.npz: rinr.net.loss_and_grad, rinr.encoder._train /
fit_round1 / fit_full).

Bars (fp32 with a different summation order, so trajectories agree
statistically, not bitwise):
  * loss_and_grad, accurate sine: loss rel <= 1e-5, per-layer gradient
    ||g - g_ref|| / ||g_ref|| <= 1e-4; MUFU sine: 2e-3 / 2e-3
  * 40 Adam steps: every sampled loss within 1e-3 relative
  * fit_round1 / fit_full (short schedules): every PSNR within 0.1 dB,
    final prune ratio equal
  * masked weights stay exactly 0; a batch fit equals per-image fits bitwise
"""

import numpy as np
import pytest
import torch

from transforms_common import split, split_bias

pytestmark = pytest.mark.gpu
DIMS = (2, 15, 15, 3)


@pytest.fixture(scope="module")
def E():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2306_16699_b200 import encoder
    return encoder


def _dm(g, key, E):
    from paper_2306_16699_b200 import synth, transforms as T
    w = torch.from_numpy(g[f"{key}/w"].astype(np.float32)[None]).cuda()
    b = torch.from_numpy(g[f"{key}/b"].astype(np.float32)[None]).cuda()
    m = torch.from_numpy(g[f"{key}/mask"][None]).cuda() if f"{key}/mask" in g else torch.ones_like(w, dtype=torch.uint8)
    return T.DeviceModels(synth.ARCH_A, w, m, b)


@pytest.mark.parametrize("sin,tol", [("accurate", (1e-5, 1e-4)), ("mufu", (2e-3, 2e-3))])
def test_loss_and_grad(golden, E, sin, tol):
    g = golden("encoder")
    for k in (0, 1):
        dm = _dm(g, f"grad{k}", E)
        img = torch.from_numpy(g["images16"][k][None]).cuda()
        loss, gw, gb = E.loss_and_grad_batch(dm, img, sin)
        assert abs(loss.item() - g[f"grad{k}/loss"]) <= tol[0] * g[f"grad{k}/loss"]
        got_w = gw[0].cpu().numpy()
        got_b = gb[0].cpu().numpy()
        for a, b in zip(split(got_w, DIMS), split(g[f"grad{k}/gw"], DIMS)):
            assert np.linalg.norm(a - b) <= tol[1] * np.linalg.norm(b), (k, sin)
        for a, b in zip(split_bias(got_b, DIMS), split_bias(g[f"grad{k}/gb"], DIMS)):
            assert np.linalg.norm(a - b) <= tol[1] * np.linalg.norm(b) + 1e-12, (k, sin)
        # masked gradient entries are exactly zero
        mask = g[f"grad{k}/mask"].astype(bool)
        assert np.all(got_w[~mask] == 0.0)


def test_train_40_steps(golden, E):
    g = golden("encoder")
    dm = E.init_batch(E.Architecture(DIMS), [33], 16, 16)
    img = torch.from_numpy(g["images16"][2][None]).cuda()
    curves, status = E.train_batch(dm, img, 5e-4, 40, "accurate")
    assert status[0] == 0
    got = curves[0][~np.isnan(curves[0])]
    want = g["train/curve"]
    assert got.shape == want.shape
    np.testing.assert_allclose(got, want, rtol=1e-3)


def test_fit_round1_and_full(golden, E):
    from paper_2306_16699_b200 import ImageBuffer
    g = golden("encoder")
    imgs = g["images32"]
    cfg1 = E.EncodeConfig(E.Architecture(DIMS), round1_steps=300, seed=int(g["round1/seed"]), sin="accurate")
    _, r1 = E.fit_round1(ImageBuffer(imgs[0]), cfg1)
    assert abs(r1.psnr_after_round[0] - g["round1/psnr"][0]) <= 0.1
    np.testing.assert_allclose(r1.loss_curve, g["round1/curve"], rtol=2e-2)
    cfgf = E.EncodeConfig(E.Architecture(DIMS), round1_steps=200, retrain_steps=100, seed=int(g["full/seed"]),
                          sin="accurate")
    model, rf = E.fit_full(ImageBuffer(imgs[1]), cfgf)
    np.testing.assert_allclose(rf.psnr_after_round, g["full/psnr"], atol=0.1)
    np.testing.assert_allclose(rf.psnr_after_mask, g["full/psnr_mask"], atol=0.1)
    assert rf.final_prune_ratio == pytest.approx(float(g["full/ratio"]), abs=1e-12)
    # pruned weights are exactly zero after retraining
    for l, m in zip(model.layers, model.mask):
        assert np.all(l.w[~m] == 0.0)


def test_batch_equals_single(golden, E):
    g = golden("encoder")
    imgs = torch.from_numpy(g["images16"]).cuda()
    dm = E.init_batch(E.Architecture(DIMS), [5, 6, 7], 16, 16)
    E.train_batch(dm, imgs, 5e-4, 25)
    for i in range(3):
        one = E.init_batch(E.Architecture(DIMS), [5 + i], 16, 16)
        E.train_batch(one, imgs[i:i + 1], 5e-4, 25)
        assert torch.equal(one.w[0], dm.w[i]) and torch.equal(one.b[0], dm.b[i])


def test_encode_dataset_roundtrip(E):
    """encode_dataset -> writer -> Store -> decode reproduces the encoder's PSNR."""
    from paper_2306_16699_b200 import Store, synth
    from paper_2306_16699_b200.archive import serialize
    from paper_2306_16699_b200.transforms import psnr
    from transforms_common import smooth_images
    x = smooth_images(4, 32, 32, seed=5)
    cfg = E.EncodeConfig(E.Architecture(DIMS), round1_steps=150, retrain_steps=60, seed=3)
    arch, rep = E.encode_dataset(list(x), cfg)
    assert len(arch.records) == 4 and not rep.failures
    data = serialize(arch)
    with Store(data) as st:
        dec = st.decode(torch.arange(4), 32, 32, layout="nhwc")
    _, p = psnr(dec, torch.from_numpy(x).cuda())
    got = p.cpu().numpy()
    want = np.array([r.psnr_after_round[-1] for r in rep.per_image])
    np.testing.assert_allclose(got, want, atol=0.05)


def test_unsupported(E):
    """Widths above 64 (the general kernel's limit) are refused; (2, 20, 20, 3)
    now runs on the general kernels."""
    from paper_2306_16699_b200 import UnsupportedError
    dm = E.init_batch(E.Architecture((2, 80, 3)), [0], 8, 8)
    with pytest.raises(UnsupportedError):
        E.train_batch(dm, torch.zeros((1, 8, 8, 3), device="cuda"), 1e-3, 2)
    dm = E.init_batch(E.Architecture((2, 20, 20, 3)), [0], 8, 8)
    curves, status = E.train_batch(dm, torch.full((1, 8, 8, 3), 0.5, device="cuda"), 1e-3, 4)
    assert status[0] == 0 and np.isfinite(curves[0][:2]).all()


@pytest.mark.parametrize("H", [8, 9, 12, 13, 14, 16])
def test_widths_vs_oracle(E, H):
    """Every supported hidden width: the first step's loss and gradients
    match the oracle's net.loss_and_grad restatement; a short fit stays finite."""
    from oracle import rinr_oracle as O
    from transforms_common import cat, smooth_images
    dims = (2, H, H, 3)
    x = smooth_images(2, 12, 20, seed=H)
    dm = E.init_batch(E.Architecture(dims), [H, H + 1], 12, 20)
    img = torch.from_numpy(x).cuda()
    loss, gw, gb = E.loss_and_grad_batch(dm, img, "accurate")
    coords = O.coordinate_grid(12, 20)
    for i in range(2):
        ws, bs, ms = O.init_model(dims, [H, H + 1][i])
        ref_loss, gws, gbs = O.loss_and_grad(ws, bs, ms, 30.0, coords, x[i].reshape(-1, 3))
        assert abs(loss[i].item() - ref_loss) <= 1e-5 * ref_loss
        a, b = gw[i].cpu().numpy(), cat(gws)
        assert np.linalg.norm(a - b) <= 1e-4 * np.linalg.norm(b)
        a, b = gb[i].cpu().numpy(), cat(gbs)
        assert np.linalg.norm(a - b) <= 1e-4 * np.linalg.norm(b) + 1e-12
    curves, status = E.train_batch(dm, img, 5e-4, 30)
    assert not status.any() and np.isfinite(curves[~np.isnan(curves)]).all()


@pytest.mark.parametrize("H,h,w", [(8, 12, 20), (11, 13, 7), (15, 32, 32), (15, 50, 44), (13, 1, 37), (14, 45, 46)])
def test_mma_pass_vs_oracle(E, H, h, w):
    """The MUFU-mode tensor-core pass (bf16 3-pass products, movmatrix
    gradient sums): loss and gradients vs the oracle at the MUFU bar (2e-3)
    for several widths, ragged sizes (partial 16-pixel tiles) and both pixel
    table modes (<= 2048 pixels cached per CTA; 50x44 and 45x46 use the
    per-axis coordinate path)."""
    from oracle import rinr_oracle as O
    from transforms_common import cat, smooth_images
    dims = (2, H, H, 3)
    x = smooth_images(2, h, w, seed=H + h)
    dm = E.init_batch(E.Architecture(dims), [H, H + 7], h, w)
    loss, gw, gb = E.loss_and_grad_batch(dm, torch.from_numpy(x).cuda(), "mufu")
    coords = O.coordinate_grid(h, w)
    for i in range(2):
        ws, bs, ms = O.init_model(dims, [H, H + 7][i])
        ref_loss, gws, gbs = O.loss_and_grad(ws, bs, ms, 30.0, coords, x[i].reshape(-1, 3))
        assert abs(loss[i].item() - ref_loss) <= 2e-3 * ref_loss, (H, h, w)
        a, b = gw[i].cpu().numpy(), cat(gws)
        assert np.linalg.norm(a - b) <= 2e-3 * np.linalg.norm(b), (H, h, w)
        a, b = gb[i].cpu().numpy(), cat(gbs)
        assert np.linalg.norm(a - b) <= 2e-3 * np.linalg.norm(b) + 1e-12, (H, h, w)
