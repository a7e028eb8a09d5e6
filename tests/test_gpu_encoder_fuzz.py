"""Randomised parity sweep of the batched GPU encoder's gradient step
(csrc/fit.cu via rinr_fit with steps = 0) against the oracle's
net.loss_and_grad restatement (net.py:217-265): random hidden widths
(8..16, so both the MMA pass and the FFMA pass), image sizes (ragged tiles,
both pixel-table modes), pruning masks, perturbed weights and biases, and
both sine modes.

Bars as stated in DESIGN.md §3.2: accurate sine, loss 1e-5 and gradient norm
1e-4 relative; MUFU sine 2e-3 / 2e-3; masked gradient entries exactly 0."""

import os

import numpy as np
import pytest
import torch

from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(int(os.environ.get("RINR_FUZZ_SEEDS", 24))))
def test_loss_and_grad_fuzz(seed):
    from paper_2306_16699_b200 import encoder as E
    from paper_2306_16699_b200 import transforms as T
    from paper_2306_16699_b200.net import Architecture
    from transforms_common import cat, smooth_images
    rng = np.random.default_rng(9000 + seed)
    H = int(rng.integers(8, 17))
    dims = (2, H, H, 3)
    h, w = (int(rng.integers(1, 60)), int(rng.integers(1, 60))) if rng.random() < 0.8 else (48, 47)
    n = int(rng.integers(1, 4))
    sin = str(rng.choice(["mufu", "accurate"]))
    x = smooth_images(n, h, w, seed=seed)
    models = []
    for i in range(n):
        ws, bs, ms = O.init_model(dims, int(rng.integers(1 << 30)))
        ws = [(wi * np.float32(rng.uniform(0.5, 2.0))).astype(np.float32) for wi in ws]
        bs = [rng.normal(0, 0.05, bi.shape).astype(np.float32) for bi in bs]
        if rng.random() < 0.6:  # a pruned model: masked weights are zero
            ms = [rng.random(m.shape) >= rng.uniform(0.0, 0.6) for m in ms]
            for m in ms:
                m.flat[int(rng.integers(m.size))] = True
            ws = [np.multiply(wi, mi).astype(np.float32) for wi, mi in zip(ws, ms)]
        models.append((ws, bs, ms))
    dm = T.DeviceModels(Architecture(dims),
                        torch.from_numpy(np.stack([cat(m[0]) for m in models])).cuda(),
                        torch.from_numpy(np.stack([cat(m[2]) for m in models]).astype(np.uint8)).cuda(),
                        torch.from_numpy(np.stack([cat(m[1]) for m in models])).cuda())
    loss, gw, gb = E.loss_and_grad_batch(dm, torch.from_numpy(x).cuda(), sin)
    tl, tg = (1e-5, 1e-4) if sin == "accurate" else (2e-3, 2e-3)
    coords = O.coordinate_grid(h, w)
    for i, (ws, bs, ms) in enumerate(models):
        ref_loss, gws, gbs = O.loss_and_grad(ws, bs, ms, 30.0, coords, x[i].reshape(-1, 3))
        ctx = (seed, H, h, w, sin, i)
        assert abs(loss[i].item() - ref_loss) <= tl * ref_loss, ctx
        a, b = gw[i].cpu().numpy(), cat(gws)
        assert np.linalg.norm(a - b) <= tg * np.linalg.norm(b), ctx
        assert np.all(a[~cat(ms)] == 0.0), ctx
        a, b = gb[i].cpu().numpy(), cat(gbs)
        assert np.linalg.norm(a - b) <= tg * np.linalg.norm(b) + 1e-12, ctx
