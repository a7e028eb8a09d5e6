"""Throughput of the batched GPU encoder (csrc/fit.cu) next to the reference
trainer's algorithm on the host cores (the oracle port of encoder._train).

    python tools/bench_encoder.py [--images 1024] [--steps 500] [--full]

Lines (JSON):
  * fit_step: images x Adam steps per second for `--steps` steps of round 1
    (CUDA events), with an FFMA-equivalent roofline over algorithmic FLOPs:
    per pixel per step forward 2*(2H + H^2 + 3H), backward deltas 2*(3H + H^2),
    weight gradients 2*(2H + H^2 + 3H) (H = 15: 1740 FLOP), against the FFMA
    peak measured by the diag microbenchmark in this process, and the MUFU
    fraction (60 sin/cos per pixel-step against the measured MUFU.SIN rate);
  * fit_full (with --full): wall-clock images/s of the whole default pipeline
    (5,000 + 10,000 + 10,000 steps, two prunes, four PSNR renders).
The CPU baseline times the oracle's numpy loss_and_grad + Adam per image on
every host core (one process each) and scales to the same step count.
"""

import argparse
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rinr_oracle as O  # noqa: E402
from paper_2306_16699_b200 import _native as N, encoder as E, synth  # noqa: E402
from transforms_common import smooth_images  # noqa: E402

H = 15
FLOP_PX = 2 * (2 * H + H * H + 3 * H) + 2 * (3 * H + H * H) + 2 * (2 * H + H * H + 3 * H)


def _cpu_worker(args):
    img, steps, seed = args
    ws, bs, ms = O.init_model((2, H, H, 3), seed)
    coords = O.coordinate_grid(img.shape[0], img.shape[1])
    t0 = time.perf_counter()
    O.train(ws, bs, ms, 30.0, coords, img.reshape(-1, 3), 5e-4, steps)
    return time.perf_counter() - t0


def cpu_rate(imgs, steps):
    cores = os.cpu_count() or 1
    with mp.get_context("fork").Pool(cores) as pool:
        t0 = time.perf_counter()
        times = pool.map(_cpu_worker, [(imgs[i % len(imgs)], steps, i) for i in range(cores)])
        wall = time.perf_counter() - t0
    per_step = float(np.mean(times)) / steps  # one image-step on one core
    return cores / per_step, cores, wall, per_step


def peaks():
    import bench
    return bench.measure_peaks(torch, N.lib())


MUFU_PX = 2 * 2 * H  # sin + cos per hidden unit of both sine layers (60 MUFU ops per pixel-step)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    n = a.images
    imgs = smooth_images(min(n, 64), 32, 32, seed=1)
    x = torch.from_numpy(imgs[np.arange(n) % len(imgs)]).cuda()
    arch = synth.ARCH_A
    seeds = [E.derive_seed(0, i) for i in range(n)]
    dm = E.init_batch(arch, seeds, 32, 32)
    E.train_batch(dm, x, 5e-4, 20)  # warm-up
    torch.cuda.synchronize()
    dm = E.init_batch(arch, seeds, 32, 32)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    curves, status = E.train_batch(dm, x, 5e-4, a.steps)
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) * 1e-3
    rate = n * a.steps / dt
    pk = peaks()
    peak = pk["ffma_flop_per_s"]
    achieved = rate * 32 * 32 * FLOP_PX
    mufu = rate * 32 * 32 * MUFU_PX
    cpu = None
    if not a.no_cpu:
        r, cores, wall, per_step = cpu_rate(imgs, 40)
        cpu = {"value": r, "unit": "image-steps/s", "cores": cores, "kind": "port",
               "sample": f"{cores} images x 40 steps of oracle encoder._train (numpy loss_and_grad + Adam, 32x32, "
                         f"arch (2,15,15,3)), one process per core, {wall:.1f} s wall; {per_step * 1e3:.2f} ms per "
                         "image-step on one core"}
    line = {"metric": "encoder image-steps/sec (full-batch Adam on 32x32, arch (2,15,15,3))", "value": rate,
            "unit": "image-steps/s", "ms": dt * 1e3, "config": {"images": n, "steps": a.steps, "h": 32, "w": 32},
            "roofline": {"bound": "ffma", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                         "frac": achieved / peak, "flop_per_pixel_step": FLOP_PX,
                         "note": "algorithmic FLOPs against the FP32 FFMA peak; in MUFU mode the products run "
                                 "as bf16 3-pass mma.sync, so this is an equivalent-throughput figure"},
            "roofline_mufu": {"bound": "mufu", "achieved": mufu / 1e12, "peak": pk["mufu_sin_per_s"] / 1e12,
                              "unit": "T op/s", "frac": mufu / pk["mufu_sin_per_s"], "ops_per_pixel_step": MUFU_PX},
            "cpu_baseline": cpu, "diverged": int((status != 0).sum()), "gpu_launches": 1}
    print(json.dumps(line), flush=True)
    if a.full:
        cfg = E.EncodeConfig(arch, seed=0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, reports, alive = E.fit_full_batch(x, cfg, seeds)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ps = np.array([r.psnr_after_round[-1] for r in reports])
        steps_total = cfg.round1_steps + 2 * cfg.retrain_steps
        full = {"metric": "encoded images/sec (full fit_full pipeline: 5000 + 10000 + 10000 Adam steps, 2 prunes)",
                "value": n / wall, "unit": "images/s", "wall_s": wall, "config": {"images": n, "h": 32, "w": 32},
                "mean_psnr_db": float(ps.mean()), "min_psnr_db": float(ps.min()),
                "mean_prune_ratio": float(np.mean([r.final_prune_ratio for r in reports]))}
        if cpu:
            full["cpu_baseline"] = dict(cpu, value=cpu["value"] / steps_total, unit="images/s",
                                        note="image-step rate / 25000 steps (training only, renders excluded)")
        print(json.dumps(full), flush=True)


if __name__ == "__main__":
    main()
