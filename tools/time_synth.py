"""Time the GPU synthetic store generator (synth.gpu_store_bytes) against the host one."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2306_16699_b200 import Store, synth  # noqa: E402

for cfg, n in (("c2", 262144), ("c3", 16384), ("c1", 262144), ("c2", 1 << 20)):
    torch.cuda.synchronize()
    t = time.perf_counter()
    data = synth.gpu_store_bytes(cfg, n, seed=1)
    t1 = time.perf_counter()
    st = Store(data)
    t2 = time.perf_counter()
    print(cfg, n, f"gen {t1 - t:.2f} s, {len(data) / 1e6:.0f} MB, store build {t2 - t1:.2f} s", flush=True)
    st.close()
