"""Affine8 hidden layers whose zero point lies outside [-1, 256].

The reference quantizer (compressor.py:175-185) gives zp = round(-min/scale),
so a layer whose kept weights all share one sign gets |zp| up to ~2^8 * max/min
(weights in [0.5, 1.0] -> zp = -255).  Then code - zp reaches 510, which bf16
cannot hold exactly; the kernels must route such layers through the float
hi/lo B split instead of the integer-code operand (device_common.cuh
int_b_exact).  fp32 decodes must stay within the 1e-3 max-abs bar and the
dequantised weights bit-exact.
"""

import numpy as np
import pytest
import torch

from conftest import bf16_bar
from oracle import rinr_oracle as O
from paper_2306_16699_b200 import synth
from paper_2306_16699_b200.compressor import quantize_batch

pytestmark = pytest.mark.gpu


def _one_signed(arch, n, seed, frac_shifted):
    """R1 random models; in a `frac_shifted` share of them every hidden layer
    is moved to one sign (all positive or all negative)."""
    mb = synth.tweak_r1(synth.random_batch(arch, n, seed))
    rng = np.random.default_rng(seed + 1)
    shifted = rng.random(n) < frac_shifted
    for l in range(1, len(arch.dims) - 2):
        w = mb.w[l]
        sign = np.where(rng.random(n) < 0.5, 1.0, -1.0).astype(np.float32)[:, None, None]
        # magnitudes in [0.1, 0.15] x max|w|: offset > spread, so zp ~ -510;
        # small enough that the 10-layer net stays well conditioned (a
        # one-signed layer at full SIREN scale amplifies f32 rounding ~15x per layer)
        mx = np.abs(w).max(axis=(1, 2), keepdims=True)
        one = (np.float32(0.1) * mx + np.float32(0.05) * np.abs(w)) * sign
        mb.w[l] = np.where(shifted[:, None, None], one, w).astype(np.float32)
    return quantize_batch(mb, "affine8"), shifted


@pytest.mark.parametrize("arch_name,size", [("A", 32), ("C", 40), ("B", 24)])
@pytest.mark.parametrize("frac", [1.0, 0.5])
def test_out_of_range_zero_point(arch_name, size, frac):
    arch = {"A": synth.ARCH_A, "B": synth.ARCH_B, "C": synth.ARCH_C}[arch_name]
    n = 24
    mb, shifted = _one_signed(arch, n, seed=7, frac_shifted=frac)
    zps = np.stack([mb.quant[l].zero_point for l in sorted(mb.quant)], 1)  # [n, hidden]
    assert np.any((zps < -1) | (zps > 256)), "the fixture must exercise out-of-range zero points"
    data = synth.archive_bytes(mb)
    models = O.read_models(data)
    from paper_2306_16699_b200 import Store
    with Store(data) as st:
        ids = torch.arange(n)
        params = st.dequantize(ids).cpu().numpy()
        for i, m in enumerate(models):
            f = O.flat_params(m)
            np.testing.assert_array_equal(params[i, :f.size].view(np.uint32), f.view(np.uint32))
        want = np.stack(O.decode_batch(models, size, size))
        for precision in ("fp32", "exact"):
            got = st.decode(ids, size, size, layout="nhwc", precision=precision).cpu().numpy()
            err = float(np.abs(got - want).max())
            assert err <= 1e-3, (precision, err)
        got = st.decode(ids, size, size, layout="nhwc", precision="bf16").cpu().numpy()
        # one-signed layers amplify rounding ~1.9x per layer (vs ~1x for SIREN
        # init), so the 10-layer nets get the bf16 bar minus 6 dB here; a
        # mis-scaled integer operand would cost tens of dB
        bar = bf16_bar(arch.dims) - (6.0 if len(arch.dims) > 4 else 0.0)
        for i in range(n):
            assert O.psnr(got[i], want[i]) >= bar, (i, bar)
