"""Full-batch accuracy of each precision mode against the CPU oracle
(run with -s to see the numbers; DESIGN.md §3 quotes them).

Stated tolerances (north_star): fp32 mode max-abs <= 1e-3; bf16 mode stated
as per-image PSNR vs the reference decode, >= 50 dB on these random-init R1
models (last layer scaled x20)."""

import numpy as np
import pytest
import torch

from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_full_batch_accuracy(cfg):
    from paper_2306_16699_b200 import Store, synth
    if cfg == "c2":
        data, hw, n = synth.archive_bytes(synth.config2(1024, seed=11)), (32, 32), 1024
    else:
        data, hw, n = synth.archive_bytes(synth.config3(4, seed=5)), (224, 224), 4
    models = O.read_models(data)
    want = np.stack(O.decode_batch(models[:n], *hw))
    with Store(data) as st:
        for prec in ("fp32", "bf16"):
            got = st.decode(torch.arange(n), *hw, layout="nhwc", precision=prec).cpu().numpy()
            ps = [O.psnr(got[i], want[i]) for i in range(n)]
            err = float(np.abs(got - want).max())
            u8 = float((O.to_u8(got) != O.to_u8(want)).mean())
            print(f"\n{cfg} {prec}: max-abs {err:.2e}, PSNR min {min(ps):.1f} / median {np.median(ps):.1f} dB, "
                  f"u8 mismatch {100 * u8:.3f}%")
            if prec == "fp32":
                assert err <= 1e-3
            else:
                assert min(ps) >= 50.0
