"""The general GPU encoder (csrc/fit_general.cu) on deep / wide nets — the
paper's Mini-ImageNet [2,40x9,3] and a 4-layer 32-wide net — against the
reference's own results (tests/golden/encoder.npz 'wgrad*', 'wtrain': rinr
net.loss_and_grad and encoder._train).

Bars, as for the narrow kernel (fp32 with a different summation order):
  * loss_and_grad, accurate sine: loss rel <= 1e-5, per-layer gradient
    ||g - g_ref|| / ||g_ref|| <= 1e-4 (MUFU sine: 2e-3 / 2e-3); masked
    gradient entries exactly 0
  * 20 Adam steps: every sampled loss within 1e-3 relative
  * fit_round1 on arch C: PSNR rises; render matches the fused decode
"""

import numpy as np
import pytest
import torch

from transforms_common import split, split_bias

pytestmark = pytest.mark.gpu
DIMS_C = (2, *[40] * 9, 3)


def _dm(g, key, dims):
    from paper_2306_16699_b200 import transforms as T
    from paper_2306_16699_b200.net import Architecture
    w = torch.from_numpy(g[f"{key}/w"].astype(np.float32)[None]).cuda()
    b = torch.from_numpy(g[f"{key}/b"].astype(np.float32)[None]).cuda()
    m = torch.from_numpy(g[f"{key}/mask"][None]).cuda()
    return T.DeviceModels(Architecture(dims), w, m, b)


@pytest.mark.parametrize("sin,tol", [("accurate", (1e-5, 1e-4)), ("mufu", (2e-3, 2e-3))])
def test_wide_loss_and_grad(golden, sin, tol):
    from paper_2306_16699_b200 import encoder as E
    g = golden("encoder")
    for k in (0, 1):
        dm = _dm(g, f"wgrad{k}", DIMS_C)
        img = torch.from_numpy(g["images12"][k][None]).cuda()
        loss, gw, gb = E.loss_and_grad_batch(dm, img, sin)
        assert abs(loss.item() - g[f"wgrad{k}/loss"]) <= tol[0] * g[f"wgrad{k}/loss"], (k, sin)
        got_w, got_b = gw[0].cpu().numpy(), gb[0].cpu().numpy()
        for l, (a, b) in enumerate(zip(split(got_w, DIMS_C), split(g[f"wgrad{k}/gw"], DIMS_C))):
            assert np.linalg.norm(a - b) <= tol[1] * np.linalg.norm(b) + 1e-12, (k, sin, l)
        for a, b in zip(split_bias(got_b, DIMS_C), split_bias(g[f"wgrad{k}/gb"], DIMS_C)):
            assert np.linalg.norm(a - b) <= tol[1] * np.linalg.norm(b) + 1e-12, (k, sin)
        mask = g[f"wgrad{k}/mask"].astype(bool)
        assert np.all(got_w[~mask] == 0.0)


def test_wide_train_20_steps(golden):
    from paper_2306_16699_b200 import encoder as E
    g = golden("encoder")
    dm = E.init_batch(E.Architecture((2, 32, 32, 32, 3)), [44], 12, 12)
    img = torch.from_numpy(g["images12"][1][None]).cuda()
    curves, status = E.train_batch(dm, img, 2e-4, 20, "accurate")
    assert status[0] == 0
    got = curves[0][~np.isnan(curves[0])]
    np.testing.assert_allclose(got, g["wtrain/curve"], rtol=1e-3)


def test_wide_fit_round1_and_render():
    """fit_round1 on the Mini-ImageNet arch over a small batch, then the
    encoder's render against the fused decode of the same (written) models."""
    from oracle import rinr_oracle as O
    from paper_2306_16699_b200 import Store, encoder as E, transforms as T
    from transforms_common import smooth_images
    imgs = torch.from_numpy(smooth_images(3, 16, 16, seed=5)).cuda()
    cfg = E.EncodeConfig(E.Architecture(DIMS_C), round1_steps=150, round1_lr=2e-4)
    dm, reports, alive = E.fit_round1_batch(imgs, cfg, seeds=[1, 2, 3])
    assert all(a is True for a in alive)
    for r in reports:
        assert len(r.loss_curve) >= 2 and r.loss_curve[-1] < r.loss_curve[0]
        assert r.psnr_after_round[0] > 12.0
    rend = E.render(dm, 16, 16, "accurate").cpu().numpy()
    data = T.serialize(dm).cpu().numpy().tobytes()
    want = np.stack(O.decode_batch(O.read_models(data), 16, 16))
    assert float(np.abs(rend - want).max()) <= 1e-4
    with Store(data) as st:
        dec = st.decode(torch.arange(3), 16, 16, layout="nhwc", precision="fp32").cpu().numpy()
    assert float(np.abs(dec - want).max()) <= 1e-3
