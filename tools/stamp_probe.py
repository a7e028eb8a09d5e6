import sys, torch
sys.path.insert(0, '/root/repo')
import bench
from paper_2306_16699_b200 import Store
st = Store(bench.store_bytes('c2', 65536, seed=0))
for B in (148, 1024, 4096):
    ids = torch.randint(0, len(st), (B,), device='cuda')
    p = st.decode_params(32, 32, precision='fp32', overlap_prologue=True)
    out = torch.empty((B, 3, 32, 32), device='cuda')
    for k in range(4):
        print(B, k, file=sys.stderr, flush=True)
        st.decode(ids, out=out, params=p, check=False)
    torch.cuda.synchronize()
