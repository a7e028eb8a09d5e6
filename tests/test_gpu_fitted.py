"""Decode parity on INRs the reference encoder actually fitted
(tests/golden/fitted.npz: encoder.fit_round1, then prune + affine8 as the
paper stores them).  The stated bar for every precision:
|PSNR(gpu decode, source) - PSNR(reference decode, source)| <= 0.05 dB per
image; fp32 / exact also max-abs <= 1e-3 against the reference decode."""

import numpy as np
import pytest
import torch

from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu

DPSNR_DB = 0.05


@pytest.mark.parametrize("name", ["A", "C"])
@pytest.mark.parametrize("precision", ["fp32", "bf16", "exact"])
def test_fitted_psnr_delta(golden, name, precision):
    from paper_2306_16699_b200 import Store
    g = golden("fitted")
    src, want, ref_psnr = g[f"{name}/source"], g[f"{name}/decode"], g[f"{name}/psnr"]
    n, h, w = src.shape[0], src.shape[1], src.shape[2]
    with Store(g[f"{name}/archive"].tobytes()) as st:
        got = st.decode(torch.arange(n), h, w, layout="nhwc", precision=precision).cpu().numpy()
    for i in range(n):
        d = abs(O.psnr(got[i], src[i]) - ref_psnr[i])
        assert d <= DPSNR_DB, (name, precision, i, d)
    if precision != "bf16":
        assert float(np.abs(got - want).max()) <= 1e-3
