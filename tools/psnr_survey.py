"""bf16-mode PSNR vs the reference decode over the golden stores and the fuzz
generator (development survey for the stated bf16 bar)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import STORE_CASES, load_golden
from oracle import rinr_oracle as O
from paper_2306_16699_b200 import Store
import test_gpu_fuzz as F

for case in STORE_CASES:
    g = load_golden(case)
    with Store(g["archive"].tobytes()) as st:
        for key in g:
            if not key.startswith("decode_"):
                continue
            h, w = map(int, key[len("decode_"):].split("x"))
            want = g[key]
            got = st.decode(torch.arange(want.shape[0]), h, w, layout="nhwc", precision="bf16").cpu().numpy()
            ps = [O.psnr(got[i], want[i]) for i in range(want.shape[0])]
            print(case, key, "min %.1f median %.1f" % (min(ps), float(np.median(ps))))
worst = []
for seed in range(200):
    rng = np.random.default_rng(1000 + seed)
    data = F._random_store(rng)
    models = O.read_models(data)
    with Store(data) as st:
        h, w = 32, 32
        ids = torch.arange(len(models))
        out = st.decode(ids, h, w, layout="nhwc", precision="bf16").cpu().numpy()
        for j, m in enumerate(models):
            worst.append((O.psnr(out[j], O.decode(m, h, w)), seed, m.layers[1].w.shape if len(m.layers) > 1 else None))
worst.sort(key=lambda t: t[0])
print("fuzz worst", worst[:8])
print("fuzz pct", np.percentile([w[0] for w in worst], [0, 1, 5, 50]))
