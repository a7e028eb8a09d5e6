"""Throughput of the GPU encoder-side transforms (csrc/transforms.cu) next to
the CPU oracle, which is the reference's per-model numpy algorithm.  Prints one
JSON line per transform.

    python tools/bench_transforms.py [--models 65536] [--arch A|C] [--reps 10]

Roofline: HBM with algorithmic bytes (weights read + written, masks, codes):
  prune_l1: 4P read + P mask read + 4P write + P mask write = 10P B per model
  quantize: 4P + P read, 4P + 2P (u16 codes) write over all matrices = 11P B
  psnr:     2 x 4 x values read
against MEASURED_PEAKS.json hbm_gbs.  The prune bisection is one CTA per
model, ~31 block-wide counting passes over the model's P keys in shared
memory.  It is bound by sync latency, not HBM; the fraction says so.
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

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rinr_oracle as O  # noqa: E402
from paper_2306_16699_b200 import synth, transforms as T  # noqa: E402


def _cpu_chunk(args):
    ws, ms, bs, ratios = args
    for w, m, b, r in zip(ws, ms, bs, ratios):
        pw, pm = O.prune_l1(w, m, float(r))
        O.quantize(pw, pm, b, 8)
    return len(ws)


def cpu_rate(mb, ratios, seconds=5.0):
    """Oracle prune + quantize per model over all host cores (fork pool)."""
    cores = os.cpu_count() or 1
    n = mb.n
    models = []
    for k in range(n):
        models.append(([w[k] for w in mb.w], [m[k] for m in mb.mask], [b[k] for b in mb.b], ratios[k]))
    # calibrate on one core
    t0 = time.perf_counter()
    _cpu_chunk(tuple(map(list, zip(*models[:32]))))
    per = (time.perf_counter() - t0) / 32
    total = max(cores, min(n, int(seconds * cores / per)))
    chunks = [tuple(map(list, zip(*[models[(i * 7) % n] for i in range(c, total, cores)]))) for c in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        t0 = time.perf_counter()
        done = sum(pool.map(_cpu_chunk, chunks))
        dt = time.perf_counter() - t0
    return done / dt, cores, done, dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", type=int, default=65536)
    ap.add_argument("--arch", default="A")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    arch = synth.ARCH_A if a.arch == "A" else synth.ARCH_C
    n = a.models if a.arch == "A" else min(a.models, 8192)
    mb = synth.tweak_r1(synth.random_batch(arch, n, seed=3))
    ratios = np.random.default_rng(4).uniform(0.05, 0.4, n)
    dm0 = T.DeviceModels.from_batch(mb)
    P = dm0.w.shape[1]
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] * 1e9
    r = torch.from_numpy(ratios).cuda()
    copies = [T.DeviceModels(dm0.arch, dm0.w.clone(), dm0.mask.clone(), dm0.b.clone()) for _ in range(a.reps + 2)]
    for c in copies[:2]:  # warm-up
        T.prune_l1(c, r, check=False)
        T.quantize(c, "affine8", check=False)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tp = tq = 0.0
    for c in copies[2:]:
        ev[0].record()
        T.prune_l1(c, r, check=False)
        ev[1].record()
        T.quantize(c, "affine8", check=False)
        ev[2].record()
        torch.cuda.synchronize()
        tp += ev[0].elapsed_time(ev[1]) * 1e-3
        tq += ev[1].elapsed_time(ev[2]) * 1e-3
    tp /= a.reps
    tq /= a.reps
    x = torch.rand((4096, 32, 32, 3), device="cuda")
    y = (x + 0.01 * torch.randn_like(x)).clamp(0, 1)
    T.psnr(x, y)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(a.reps):
        T.psnr(x, y)
    ev[1].record()
    torch.cuda.synchronize()
    ts = ev[0].elapsed_time(ev[1]) * 1e-3 / a.reps
    cpu = None
    if not a.no_cpu:
        rate, cores, done, dt = cpu_rate(mb, ratios)
        cpu = {"value": rate, "unit": "models/s", "cores": cores, "kind": "port",
               "sample": f"{done} arch-{a.arch} models, oracle prune_l1 + quantize(affine8) per model "
                         f"(compressor.py:108-202), {cores} processes, {dt:.1f} s wall"}
    for name, t, byts, unit_n in (("prune_l1", tp, 10 * P, n), ("quantize_affine8", tq, 11 * P, n),
                                  ("psnr_32x32", ts, 2 * 4 * 32 * 32 * 3, 4096)):
        line = {"metric": f"{name} models/sec" if name != "psnr_32x32" else "psnr images/sec",
                "value": unit_n / t, "unit": "models/s" if name != "psnr_32x32" else "images/s",
                "config": {"arch": list(arch.dims), "models": unit_n, "params_per_model": P},
                "ms": t * 1e3,
                "roofline": {"bound": "hbm", "achieved": byts * unit_n / t / 1e9, "peak": peak / 1e9,
                             "unit": "GB/s", "frac": byts * unit_n / t / peak},
                "gpu_launches": 1}
        if cpu and name == "quantize_affine8":
            line["cpu_baseline_prune_plus_quantize"] = cpu
            line["gpu_prune_plus_quantize_models_per_s"] = n / (tp + tq)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
