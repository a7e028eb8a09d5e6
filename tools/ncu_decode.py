"""Fixed-launch decode driver for ncu captures (never used for bench numbers).

    python tools/ncu_decode.py --config c2 --launches 20
    ncu --set full -k regex:decode_mma -s 5 -c 1 -o prof python tools/ncu_decode.py ...
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_16699_b200 import Store  # noqa: E402
from paper_2306_16699_b200.store import IMAGENET_MEAN, IMAGENET_STD, resized_crop_params  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--launches", type=int, default=20)
    ap.add_argument("--records", type=int, default=65536)
    ap.add_argument("--precision", default=None)
    ap.add_argument("--batch", type=int, default=None)
    a = ap.parse_args()
    W = bench.workload(a.config)
    from paper_2306_16699_b200 import synth
    st = Store(synth.gpu_store_bytes(a.config, a.records, seed=0))
    B, H, Wd = a.batch or W["batch"], W["h"], W["w"]
    ids = torch.randint(0, len(st), (a.launches, B), device="cuda")
    prec = a.precision or ("bf16" if a.config == "c3" else "fp32")
    if a.config == "c3":
        aug = resized_crop_params(B, generator=torch.Generator().manual_seed(0)).cuda()
        p = st.decode_params(H, Wd, dtype=torch.bfloat16, precision=prec, aug_mode="crop", mean=IMAGENET_MEAN,
                             std=IMAGENET_STD)
        out = torch.empty((B, 3, H, Wd), dtype=torch.bfloat16, device="cuda")
    else:
        aug = None
        p = st.decode_params(H, Wd, precision=prec)
        out = torch.empty((B, 3, H, Wd), device="cuda")
    for k in range(a.launches):
        st.decode(ids[k], out=out, aug=aug, params=p, check=False)
    torch.cuda.synchronize()
    print("ok", a.config, a.launches)


if __name__ == "__main__":
    main()
