"""CPU checks of the encoder host logic: seeds, LR schedule and config
validation mirror rinr.encoder (golden: tests/golden/encoder.npz)."""

import math

import numpy as np
import pytest

from paper_2306_16699_b200 import InvalidInputError, synth
from paper_2306_16699_b200.compressor import dynamic_ratio, get_schedule


def test_derive_seed_golden(golden):
    from paper_2306_16699_b200.encoder import derive_seed
    g = golden("encoder")
    got = [derive_seed(s, i) for s in (0, 7, 2 ** 40) for i in (0, 1, 999)]
    np.testing.assert_array_equal(np.array(got, np.uint64), g["derive_seed"])
    assert int(g["round1/seed"]) == derive_seed(7, 0) and int(g["full/seed"]) == derive_seed(7, 1)


def test_cosine_and_config():
    from paper_2306_16699_b200.encoder import EncodeConfig, cosine_lr
    assert cosine_lr(1.0, 0, 10) == 1.0 and cosine_lr(1.0, 10, 10) == 0.0
    assert math.isclose(cosine_lr(5e-4, 5, 10), 2.5e-4)
    for bad in (dict(round1_steps=0), dict(retrain_lr=0.0), dict(iterative_prune_ratio=1.0), dict(schedule="x"),
                dict(sin="poly")):
        with pytest.raises(InvalidInputError):
            EncodeConfig(synth.ARCH_A, **bad)
    assert dynamic_ratio(get_schedule("cifar"), 32.0) == 0.05 * 32.0 - 1.5
