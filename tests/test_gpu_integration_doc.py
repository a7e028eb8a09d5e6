"""The ctypes stubs shown in INTEGRATION.md run as written (the C ABI a
reference maintainer would bind, without this repo's Python package)."""

import re
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _blocks():
    return re.findall(r"```python\n(.*?)```", (ROOT / "INTEGRATION.md").read_text(), re.S)


def test_encoder_side_stub_runs(monkeypatch):
    monkeypatch.chdir(ROOT)
    code = [b for b in _blocks() if "rinr_prune_l1.argtypes" in b]
    assert len(code) == 1
    env = {"n": 64}
    exec(compile(code[0], "INTEGRATION.md", "exec"), env)
    w, mask = env["w"], env["mask"]
    assert int((mask == 0).sum()) == 64 * 60  # k = floor(0.2 * 300 + 0.5) per model
    assert bool(((w == 0) | (mask == 1)).all())


def test_decode_stub_runs(monkeypatch, tmp_path):
    """Section 2's torch-free stub, with the archive path pointed at a
    synthetic c2 archive and the caller-filled ids set to record 0."""
    import ctypes as C

    import numpy as np
    import torch
    from paper_2306_16699_b200 import Store, synth
    monkeypatch.chdir(ROOT)
    arc = tmp_path / "train.rinr"
    arc.write_bytes(synth.archive_bytes(synth.config2(8, seed=3)))
    code = [b for b in _blocks() if "rinr_decode.argtypes" in b]
    assert len(code) == 1
    src = code[0].replace('"train.rinr"', repr(str(arc)))
    src = src.replace("_, d_ids = rt.cudaMalloc(8 * n)", "_, d_ids = rt.cudaMalloc(8 * n); rt.cudaMemset(d_ids, 0, 8 * n)")
    env = {}
    exec(compile(src, "INTEGRATION.md", "exec"), env)
    rt = env["rt"]
    n, H, W = env["n"], env["H"], env["W"]
    host = np.empty((n, 3, H, W), np.float32)
    rt.cudaDeviceSynchronize()
    rt.cudaMemcpy(host.ctypes.data, env["d_out"], host.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    with Store(arc.read_bytes()) as st:
        want = st.decode(torch.zeros(1, dtype=torch.int64), H, W).cpu().numpy()[0]
    assert np.array_equal(host[0], want) and np.array_equal(host[n - 1], want)
    env["lib"].rinr_store_destroy.argtypes = [C.c_void_p]
    env["lib"].rinr_store_destroy(env["store"])
    rt.cudaFree(env["d_ids"])
    rt.cudaFree(env["d_out"])


def test_writer_stub_runs(monkeypatch):
    """Section 2b's writer stub produces the reference writer's bytes."""
    import torch
    from paper_2306_16699_b200 import synth, transforms as T
    from paper_2306_16699_b200.archive import serialize_batch
    monkeypatch.chdir(ROOT)
    mb = synth.config1(16)
    mb.source_h, mb.source_w = 32, 32
    dm = T.DeviceModels.from_batch(mb)
    code = [b for b in _blocks() if "rinr_serialize_size.argtypes" in b]
    assert len(code) == 1
    env = {"w": dm.w, "mask": dm.mask, "b": dm.b}
    exec(compile(code[0], "INTEGRATION.md", "exec"), env)
    torch.cuda.synchronize()
    assert env["data"] == serialize_batch(dm.to_batch(), [f"img{i:08d}" for i in range(16)])
