"""Development probe: decode time vs batch size (fixed cost vs per-image cost).

    python tools/scale_probe.py --config c2 --batches 128,256,512,1024,2048,4096
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
    ap.add_argument("--batches", default="128,256,512,1024,2048,4096")
    ap.add_argument("--records", type=int, default=65536)
    ap.add_argument("--precision", default=None)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--overlap", action="store_true")
    a = ap.parse_args()
    W = bench.workload(a.config)
    st = Store(bench.store_bytes(a.config, a.records, seed=0))
    H, Wd = W["h"], W["w"]
    prec = a.precision or ("bf16" if a.config == "c3" else "fp32")
    for B in [int(x) for x in a.batches.split(",")]:
        ids = torch.randint(0, len(st), (a.reps, B), device="cuda")
        if a.config == "c3":
            aug = resized_crop_params(B, generator=torch.Generator().manual_seed(0)).cuda()
            p = st.decode_params(H, Wd, dtype=torch.bfloat16, precision=prec, aug_mode="crop", mean=IMAGENET_MEAN,
                                 std=IMAGENET_STD, overlap_prologue=a.overlap)
            out = torch.empty((B, 3, H, Wd), dtype=torch.bfloat16, device="cuda")
        else:
            aug = None
            p = st.decode_params(H, Wd, precision=prec, overlap_prologue=a.overlap)
            out = torch.empty((B, 3, H, Wd), device="cuda")
        for k in range(3):
            st.decode(ids[k], out=out, aug=aug, params=p, check=False)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for k in range(a.reps):
                st.decode(ids[k], out=out, aug=aug, params=p, check=False)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.reps
        print(f"{a.config} {prec} ov={int(a.overlap)} batch {B:6d}: {us:9.2f} us/launch  {B / us:8.3f} Mimg/s  {us / B * 1e3:8.3f} ns/img",
              flush=True)


if __name__ == "__main__":
    main()
