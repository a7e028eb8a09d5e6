"""Throughput of the general GPU encoder (fit_general.cu) on the paper's wide
nets: Adam image-steps/s and the FFMA rate at ~6 FLOP per weight per pixel
(forward, delta and weight-gradient products)."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2306_16699_b200 import encoder as E  # noqa: E402
from paper_2306_16699_b200.net import Architecture  # noqa: E402
sys.path.insert(0, "tests")
from transforms_common import smooth_images  # noqa: E402


def run(dims, n, size, steps):
    arch = Architecture(dims)
    imgs = torch.from_numpy(smooth_images(n, size, size, seed=1)).cuda()
    dm = E.init_batch(arch, list(range(n)), size, size)
    E.train_batch(dm, imgs, 1e-4, 2)  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    E.train_batch(dm, imgs, 1e-4, steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    P = sum(a * b for a, b in zip(dims[:-1], dims[1:]))
    flop = 6.0 * P * size * size * n * steps
    return {"dims": f"[2,{dims[1]}x{len(dims) - 2},3]", "images": n, "size": size, "steps": steps,
            "image_steps_per_s": n * steps / dt, "tflops_ffma_equiv": flop / dt / 1e12, "s": round(dt, 3)}


if __name__ == "__main__":
    sys.path.insert(0, "tests")
    for dims, n, size, steps in (((2, *[40] * 9, 3), 64, 32, 50), ((2, *[40] * 9, 3), 8, 224, 10),
                                 ((2, *[32] * 9, 3), 64, 32, 50)):
        print(json.dumps(run(dims, n, size, steps)), flush=True)
