"""The GPU bench harness (harness.bench, rinr.bench.bench's mirror) against
the reference harness's own digests (tests/golden/digests.npz, made by
running rinr.bench.bench): sha256 over the decoded u8 pixels in record order.
Every record's GPU u8 pixels (precision 'exact', accurate sine) hash
identically to the reference's decoder.decode(...).as_u8(), and the
whole-archive digest equals the reference harness's (measured on B200 for all
five stores)."""

import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
CASES = ["c1_r0", "c1_r1", "c2", "zoo", "fitted_A"]


def _archive(golden, case):
    if case == "fitted_A":
        return golden("fitted")["A/archive"].tobytes()
    return golden(case)["archive"].tobytes()


@pytest.mark.parametrize("case", CASES)
def test_digest_vs_reference(golden, case):
    from paper_2306_16699_b200 import Store, bench
    g = golden("digests")
    data = _archive(golden, case)
    want_per = [str(x) for x in g[f"{case}/per_record"]]
    got_per = []
    with Store(data) as st:
        for k in range(len(st)):
            m = st.record_meta(k)
            u8 = st.decode(torch.tensor([k]), m["source_h"], m["source_w"], dtype=torch.uint8, layout="nhwc",
                           precision="exact", sin="accurate").cpu().numpy()[0]
            got_per.append(hashlib.sha256(u8.tobytes()).hexdigest())
    assert got_per == want_per, case
    assert bench(data, batch=4).digest == str(g[f"{case}/digest"]), case
