"""RINR_FLAG_PREFETCH_NEXT (Store.decode(..., next_ids=...)): the next
batch's record slots are prefetched into L2; the decoded images must be
bit-identical to a decode without it, for adjacent (zero-copy) and separate
next-id tensors, out-of-range next ids (skipped, no status), every precision,
and both kernels (narrow c2 nets and the tcgen05 wide-net kernel, which
ignores the flag)."""

import numpy as np
import pytest
import torch

from oracle import rinr_oracle as O
from paper_2306_16699_b200.errors import InvalidInputError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    from paper_2306_16699_b200 import Store, synth
    data = synth.archive_bytes(synth.config2(300, seed=11))
    st = Store(data)
    yield st, O.read_models(data)
    st.close()


@pytest.mark.parametrize("precision", ["fp32", "bf16", "exact"])
def test_prefetch_bit_identical(c2, precision):
    st, models = c2
    g = torch.Generator(device="cuda").manual_seed(3)
    rows = torch.randint(0, len(st), (3, 257), device="cuda", generator=g)
    want = st.decode(rows[0], 32, 32, precision=precision)
    adj = st.decode(rows[0], 32, 32, precision=precision, next_ids=rows[1])
    sep = st.decode(rows[0], 32, 32, precision=precision, next_ids=rows[2].clone())
    assert torch.equal(want, adj) and torch.equal(want, sep)
    if precision == "fp32":
        i = int(rows[0, 5])
        assert float(np.abs(want[5].permute(1, 2, 0).cpu().numpy() - O.decode(models[i], 32, 32)).max()) <= 1e-3


def test_prefetch_graph_steps(c2):
    """The bench pattern: K steps captured in a CUDA graph, step k passing row k+1."""
    st, _ = c2
    K, B = 6, 512
    ids = torch.randint(0, len(st), (K + 1, B), device="cuda", generator=torch.Generator(device="cuda").manual_seed(9))
    p = st.decode_params(32, 32, overlap_prologue=True, prefetch_next=True)
    outs = [torch.empty((B, 3, 32, 32), device="cuda") for _ in range(K)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        st.decode(ids[0], out=outs[0], params=p, check=False, next_ids=ids[1])
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for k in range(K):
            st.decode(ids[k], out=outs[k], params=p, check=False, next_ids=ids[k + 1])
    graph.replay()
    torch.cuda.synchronize()
    for k in range(K):
        assert torch.equal(outs[k], st.decode(ids[k], 32, 32))


def test_prefetch_bad_next_ids_ignored(c2):
    st, _ = c2
    ids = torch.arange(64, device="cuda")
    nxt = torch.full((64,), 10 ** 9, dtype=torch.int64, device="cuda")
    nxt[::2] = -5
    assert torch.equal(st.decode(ids, 32, 32), st.decode(ids, 32, 32, next_ids=nxt))  # check=True: no status raised


def test_prefetch_argument_errors(c2):
    st, _ = c2
    ids = torch.arange(8, device="cuda")
    with pytest.raises(InvalidInputError):
        st.decode(ids, 32, 32, next_ids=torch.arange(7, device="cuda"))
    p = st.decode_params(32, 32, prefetch_next=True)
    with pytest.raises(InvalidInputError):
        st.decode(ids, params=p)


def test_prefetch_wide_net_kernel():
    from paper_2306_16699_b200 import Store, synth
    data = synth.archive_bytes(synth.config3(24, seed=2))
    with Store(data) as st:
        ids = torch.arange(24, device="cuda").flip(0)
        a = st.decode(ids[:12], 64, 64, precision="bf16")
        b = st.decode(ids[:12], 64, 64, precision="bf16", next_ids=ids[12:])
        assert torch.equal(a, b)
