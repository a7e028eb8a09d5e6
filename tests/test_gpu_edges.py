"""Edge cases of the Store.decode / rinr_decode boundary: empty and
single-pixel outputs, very large batches, repeated ids, ids given as CPU
tensors / lists / int32, and out-of-range ids anywhere in a large batch."""

import numpy as np
import pytest
import torch

from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    from paper_2306_16699_b200 import Store, synth
    data = synth.archive_bytes(synth.config2(64, seed=5))
    st = Store(data)
    yield st, O.read_models(data)
    st.close()


def test_empty_batch(c2):
    st, _ = c2
    out = st.decode(torch.zeros(0, dtype=torch.int64), 32, 32)
    assert out.shape == (0, 3, 32, 32)


def test_one_pixel_and_thin_outputs(c2):
    st, models = c2
    for h, w in ((1, 1), (1, 64), (64, 1), (3, 2)):
        got = st.decode(torch.arange(8), h, w, layout="nhwc").cpu().numpy()
        for i in range(8):
            assert float(np.abs(got[i] - O.decode(models[i], h, w)).max()) <= 1e-3


def test_ids_forms_and_repeats(c2):
    st, models = c2
    want = st.decode(torch.tensor([3, 3, 7, 0]), 32, 32).cpu()
    for ids in ([3, 3, 7, 0], np.array([3, 3, 7, 0], np.int32), torch.tensor([3, 3, 7, 0], dtype=torch.int32),
                torch.tensor([0, 3, 9, 3, 11, 7, 5, 0])[[1, 3, 5, 0]]):
        assert torch.equal(st.decode(ids, 32, 32).cpu(), want)
    assert torch.equal(want[0], want[1])


def test_large_batch_matches_small(c2):
    """65,536 ids (many images per CTA, several phase-1 chunks): every image
    equals its decode in a 1-image batch (bitwise, same kernels)."""
    st, _ = c2
    g = torch.Generator().manual_seed(0)
    ids = torch.randint(0, 64, (65536,), generator=g)
    out = st.decode(ids, 32, 32)
    single = st.decode(torch.arange(64), 32, 32)
    for pos in (0, 1, 12345, 40000, 65535):
        assert torch.equal(out[pos], single[int(ids[pos])])


def test_bad_id_in_large_batch(c2):
    from paper_2306_16699_b200 import BatchItemError
    st, _ = c2
    ids = torch.randint(0, 64, (20000,))
    ids[15000] = 64
    ids[17000] = -5
    with pytest.raises(BatchItemError) as e:
        st.decode(ids, 32, 32)
    assert e.value.index == 15000


def test_store_default_device_is_current_device():
    """Store(device='cuda') lands on torch's current device."""
    import torch
    from paper_2306_16699_b200 import Store, synth
    torch.cuda.set_device(0)
    with Store(synth.archive_bytes(synth.config2(4, seed=1)), device="cuda") as st:
        assert st.device.index == torch.cuda.current_device()
        out = st.decode(torch.arange(4), 8, 8)
        assert out.device == st.device


def test_round2_prune_failure_is_per_image():
    """A prune that would empty a layer fails that image alone (StructuralError
    under on_error='skip'); the others are pruned (encoder.py:120-135)."""
    import numpy as np
    import torch
    from paper_2306_16699_b200 import StructuralError, encoder, synth, transforms as T
    mb = synth.tweak_r1(synth.random_batch(synth.ARCH_A, 3, seed=2))
    dm = T.DeviceModels.from_batch(mb)
    # model 1: layer 0 (30 weights) keeps a single, tiny weight -> a 0.5 global
    # prune empties layer 0 for it only
    m0 = dm.mask[1, :30].clone()
    m0[:] = 0
    m0[0] = 1
    dm.mask[1, :30] = m0
    dm.w[1, :30] = dm.w[1, :30] * m0.float()
    dm.w[1, 0] = 1e-6
    alive = [True, True, True]
    encoder._prune_round(dm, 0.5, alive, "skip")
    assert alive[0] is True and alive[2] is True
    assert isinstance(alive[1], StructuralError)
    keep = dm.mask.cpu().numpy().sum(axis=1)
    assert keep[0] < 300 and keep[2] < 300
    with pytest.raises(Exception):
        encoder._prune_round(dm, 0.5, [True, True, True], "fail_fast")
