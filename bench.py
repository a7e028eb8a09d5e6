#!/usr/bin/env python
"""Decode throughput bench (BASELINE.json metric: decoded images/sec, 32x32
and 224x224, % of the MUFU roofline).

Default run (`python bench.py [--gpus N --steps K --warmup W]`): ONE JSON
line whose headline is BASELINE configs[1] (c2), with the other two decode
configs of the metric as sub-objects carrying the same keys:
  c2 (headline): batch 1024, 32x32, arch [2,15,15,3], records R1-initialised,
      L1-pruned to a per-record dynamic ratio (mean ~15%) and affine8-
      quantised; fp32 NCHW out, precision 'fp32' (bf16x3 tensor-core split,
      max-abs <= 1e-3 vs the reference).
  "c1": configs[0], the reference's own CPU case: batch 256, 32x32, fp32
      dense random-init (R1) records.
  "c3": configs[2]: batch 256 of arch [2,40x9,3] (affine8, 25% pruned) at
      224x224 with random-resized-crop + flip + ImageNet normalise, bf16 NCHW
      out; credited at precision 'fp32' (bf16x3), precision 'bf16' beside it.
Every store is larger than the 126 MB L2 (c2 262,144 records = 208 MB, c1
262,144 = 366 MB, c3 16,384 = 223 MB per GPU) and every step decodes a fresh
random batch of ids, so the records a step reads are not L2-resident.  The
stores are generated on the GPU (synth.gpu_store_bytes: init + prune +
quantize + the byte-exact GPU writer) and loaded through the public Store.

A step = one fused decode launch over one batch (record fetch + bit-exact
dequant prologue + MLP + epilogue).  `value` is device throughput with ids
resident in HBM: CUDA events around one CUDA-graph replay of exactly --steps
launches, after --warmup steps and ~0.5 s of replays that keep the clocks at
their loaded state, max over ranks.  `e2e` runs the same steps through the
public API with host buffers (per step: H2D of the ids from pinned memory,
decode, D2H of the ImageBuffer-layout NHWC f32 batch).  `e2e_dropin` (c2)
times the reference-API drop-in rinr.decode_batch(models, 32, 32) on host
InrModels (serialise + store + decode + ImageBuffers).

`--impl reference` times the reference algorithm on the host CPU instead
(the numpy oracle port of rinr.decode_batch, oracle/rinr_oracle.py — the
reference package is pure Python and cannot travel to the GPU box), one
worker process per core, on the same configs.

Multi-GPU (torchrun, one process per GPU): every rank generates the same
world x R record archive and opens its shard with Store(..., shard_rank,
shard_world) (records k % world == rank); each rank decodes its own batches
with no collective (scaling "weak"); the barrier and the max-over-ranks
timing reduction are the only NCCL calls.  `--config c4` / `c5`: ResNet-18
training fed by the decode (c5: 1,048,576-record store sharded over the
ranks, DDP gradient all-reduce over NCCL).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # CPU legs: one BLAS thread per worker process

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HIDDEN_SUM = {"c1": 30, "c2": 30, "c3": 360}


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c1", "c2", "c3", "c4", "c5"], default="c2")
    ap.add_argument("--precision", choices=["fp32", "bf16", "exact"], default=None)
    ap.add_argument("--store-records", type=int, default=None, help="records per GPU")
    ap.add_argument("--no-subs", action="store_true", help="headline config only (no c1 / c3 sub-objects)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="do not let a decode's prologue overlap the previous decode (PDL off)")
    ap.add_argument("--no-prefetch", action="store_true",
                    help="do not pass the next step's ids (no L2 prefetch of the next batch's records)")
    return ap.parse_args(argv)


def workload(cfg: str):
    if cfg == "c4":
        return dict(batch=64, h=224, w=224, arch=[2] + [40] * 9 + [3], records=16384, classes=10, synth="c3",
                    desc=("c4: ResNet-18 (10 classes) training step (SGD lr 1e-2 momentum 0.9, wd 5e-4, bf16 "
                          "autocast, channels_last; PAPER.md:446) fed by on-the-fly decode of 64 affine8+25%-pruned "
                          "[2,40x9,3] records per GPU at 224x224 with random-resized-crop+flip+ImageNet normalise "
                          "(bf16 NCHW)"))
    if cfg == "c5":
        return dict(batch=128, h=32, w=32, arch=[2, 15, 15, 3], records=1 << 20, classes=10, synth="c2",
                    desc=("c5: 1,048,576-record c2-style [2,15,15,3] store sharded over the GPUs (k % world), "
                          "per-GPU decode of 128 records at 32x32 with CIFAR pad-4 crop+flip+normalise (bf16 NCHW) "
                          "feeding ResNet-18 (10 classes, SGD lr 1e-2 momentum 0.9, wd 5e-4, bf16 autocast; "
                          "PAPER.md:446), DDP gradient all-reduce over NCCL"))
    if cfg == "c1":
        return dict(batch=256, h=32, w=32, arch=[2, 15, 15, 3], records=262144, desc=(
            "c1: fp32 dense [2,15,15,3] random-init (R1) records, batch 256, 32x32, fp32 NCHW out"))
    if cfg == "c2":
        return dict(batch=1024, h=32, w=32, arch=[2, 15, 15, 3], records=262144, desc=(
            "c2: quantised(affine8)+pruned(mean~15%) [2,15,15,3] records, batch 1024, 32x32, fp32 NCHW out"))
    return dict(batch=256, h=224, w=224, arch=[2] + [40] * 9 + [3], records=16384, desc=(
        "c3: affine8 + 25%-pruned [2,40x9,3] records, batch 256, 224x224, random-resized-crop+flip+ImageNet "
        "normalise, bf16 NCHW out"))


def host_store_bytes(cfg: str, n: int, seed: int) -> bytes:
    """Small stores for the CPU legs (built before CUDA is initialised)."""
    from paper_2306_16699_b200 import synth
    if cfg == "c1":
        return synth.archive_bytes(synth.tweak_r1(synth.random_batch(synth.ARCH_A, n, seed)))
    return synth.large_store_bytes(cfg, n, seed=seed)


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm (oracle port) in a process pool
# ---------------------------------------------------------------------------
_W = {}


def _cpu_init(data: bytes, out_h: int, out_w: int):
    from oracle import rinr_oracle as O
    _W["models"] = O.read_models(data)  # materialised outside the timed region, like rinr.bench (bench.py:52-54)
    _W["hw"] = (out_h, out_w)
    _W["O"] = O


def _cpu_decode(ids):
    O = _W["O"]
    h, w = _W["hw"]
    models = _W["models"]
    out = O.decode_batch([models[i] for i in ids], h, w)
    return len(out)


def _cpu_aug_decode(args):
    ids, params = args
    O = _W["O"]
    h, w = _W["hw"]
    from paper_2306_16699_b200.store import IMAGENET_MEAN, IMAGENET_STD
    for i, p in zip(ids, params):
        O.decode_augmented(_W["models"][i], h, w, O.AUG_CROP, p, IMAGENET_MEAN, IMAGENET_STD)
    return len(ids)


class CpuPool:
    def __init__(self, data: bytes, h: int, w: int, cores: int):
        import multiprocessing as mp
        self.cores = cores
        ctx = mp.get_context("fork")
        self.pool = ctx.Pool(cores, initializer=_cpu_init, initargs=(data, h, w))

    def run(self, ids: np.ndarray, aug=None) -> float:
        """Decode `ids` split across the workers; returns wall seconds."""
        parts = np.array_split(ids, self.cores)
        t0 = time.perf_counter()
        if aug is None:
            n = sum(self.pool.map(_cpu_decode, [p.tolist() for p in parts if len(p)]))
        else:
            aparts = np.array_split(aug, self.cores)
            n = sum(self.pool.map(_cpu_aug_decode, [(p.tolist(), a) for p, a in zip(parts, aparts) if len(p)]))
        assert n == len(ids)
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def crop_params_np(n: int, seed: int) -> np.ndarray:
    import torch
    from paper_2306_16699_b200.store import resized_crop_params
    return resized_crop_params(n, generator=torch.Generator().manual_seed(seed)).numpy()


def cpu_measure(cfg: str, W: dict, steps: int = None):
    """Time the reference algorithm on the host cores.  Returns
    (images/s, sample description, cores, per-step times)."""
    cores = host_cores()
    n_rec = 4096 if cfg != "c3" else 64
    data = host_store_bytes(cfg, n_rec, seed=12345)
    pool = CpuPool(data, W["h"], W["w"], cores)
    rng = np.random.default_rng(0)
    B = W["batch"]
    try:
        # calibrate: one warm batch
        ids = rng.integers(0, n_rec, B if cfg != "c3" else cores)
        aug = crop_params_np(len(ids), 0) if cfg == "c3" else None
        pool.run(ids, aug)
        times = []
        if steps is None:  # bounded sample: ~10-30 s of CPU work across the cores
            n = min(262144, cores * 8192) if cfg == "c2" else (min(65536, cores * 2048) if cfg == "c1" else cores * 8)
            ids = rng.integers(0, n_rec, n)
            aug = crop_params_np(n, 1) if cfg == "c3" else None
            t = pool.run(ids, aug)
            sample = (f"{n} images of {cfg} ({W['h']}x{W['w']}) decoded by the oracle port of rinr.decode_batch "
                      f"(net.forward + clip{' + crop/flip/normalise' if cfg == 'c3' else ''}) from pre-materialised "
                      f"models, {cores} worker processes x 1 BLAS thread, {t:.2f} s wall")
            return n / t, sample, cores, [t]
        nb = B if cfg != "c3" else max(cores, 16)
        for _ in range(steps):
            ids = rng.integers(0, n_rec, nb)
            aug = crop_params_np(nb, len(times)) if cfg == "c3" else None
            times.append(pool.run(ids, aug))
        sample = (f"per step {nb} images of {cfg} ({W['h']}x{W['w']}) decoded by the oracle port of "
                  f"rinr.decode_batch from pre-materialised models, {cores} worker processes x 1 BLAS thread")
        return nb * len(times) / sum(times), sample, cores, times
    finally:
        pool.close()


def reference_entry(cfg: str, args, steps: int, warmup: int) -> dict:
    W = workload(cfg)
    _, sample, cores, times = cpu_measure(cfg, W, steps=warmup + steps)
    t = sum(times[warmup:])
    per_step = W["batch"] if cfg != "c3" else max(cores, 16)
    value = per_step * steps / t
    return {
        "value": value, "unit": "images/s", "ms_per_step": 1e3 * t / steps, "steps": steps, "warmup": warmup,
        "dtype": "f32", "config": {"workload": W["desc"], "cpu": cpu_model()},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    head = reference_entry(args.config, args, args.steps, args.warmup)
    line = {"impl": "reference", "metric": "decoded images/sec", "value": head["value"], "unit": "images/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": head["config"], "cpu_baseline": head["cpu_baseline"], "e2e": head["e2e"]}
    if args.config == "c2" and not args.no_subs:
        # the other legs of the metric, a few steps each (c3: ~0.1 s per 224^2 image per core)
        line["c1"] = reference_entry("c1", args, min(args.steps, 10), min(args.warmup, 2))
        line["c3"] = reference_entry("c3", args, min(args.steps, 3), 1)
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measure_peaks(torch, lib):
    """MUFU sin/s, FFMA flop/s and mma.sync bf16 flop/s on this GPU."""
    import ctypes as C
    sink = torch.zeros(1, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {}
    for kind, name, threads, iters in ((0, "mufu_sin_per_s", 512, 4096), (1, "ffma_flop_per_s", 512, 8192),
                                       (2, "hmma_bf16_flop_per_s", 256, 2048)):
        ops = C.c_double()
        blocks = sms * 4
        for _ in range(3):
            lib.rinr_diag_launch(kind, blocks, threads, iters, C.c_void_p(sink.data_ptr()), C.c_void_p(stream),
                                 C.byref(ops))
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.rinr_diag_launch(kind, blocks, threads, iters, C.c_void_p(sink.data_ptr()), C.c_void_p(stream),
                                 C.byref(ops))
            e1.record()
            torch.cuda.synchronize()
            best = max(best, ops.value / (e0.elapsed_time(e1) * 1e-3))
        out[name] = best
    return out


def reduce_max(x: float, dist=None, device=None) -> float:
    """Max over ranks (timing is the slowest rank's; one process per GPU)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        return {}


def load_traffic(cfg, precision):
    """ncu DRAM bytes per launch of the config's decode kernel (profiles/)."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
        e = d.get(f"{cfg}_{precision}") or d.get(cfg) or {}
        return e.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def open_store(torch, cfg: str, W: dict, R: int, rank: int, world: int, local: int):
    """Every rank generates the same world x R archive on its GPU and keeps
    its shard (records k % world == rank) through the public Store."""
    from paper_2306_16699_b200 import Store, synth
    t0 = time.perf_counter()
    data = synth.gpu_store_bytes(W.get("synth", cfg), R * world, seed=4242, device=f"cuda:{local}")
    st = Store(data, device=f"cuda:{local}", shard_rank=rank, shard_world=world)
    del data
    torch.cuda.synchronize()
    return st, time.perf_counter() - t0


def measure_decode(torch, dist, cfg: str, precision: str, args, rank: int, world: int, local: int, peaks: dict,
                   st=None, build_s=None, with_e2e: bool = True) -> dict:
    """One decode config on this rank's GPU: graph-timed value, roofline,
    clocks and (optionally) e2e through the public API."""
    from paper_2306_16699_b200.store import IMAGENET_MEAN, IMAGENET_STD, resized_crop_params
    from paper_2306_16699_b200.trace import stage
    W = workload(cfg)
    R = args.store_records if (args.store_records and cfg == args.config) else W["records"]
    own = st is None
    if own:
        st, build_s = open_store(torch, cfg, W, R, rank, world, local)
    B, H, Wd = W["batch"], W["h"], W["w"]
    K, Wu = args.steps, args.warmup
    gen = torch.Generator(device="cuda").manual_seed(1 + rank)
    # one spare row: step k passes row k+1 as next_ids (L2 prefetch of the next batch's records)
    ids = torch.randint(0, len(st), (Wu + K + 1, B), device="cuda", generator=gen, dtype=torch.int64)
    pf = not args.no_prefetch
    if cfg == "c3":
        aug = [resized_crop_params(B, generator=torch.Generator().manual_seed(1000 * rank + s)).cuda()
               for s in range(Wu + K)]
        params = st.decode_params(H, Wd, dtype=torch.bfloat16, precision=precision, aug_mode="crop",
                                  mean=IMAGENET_MEAN, std=IMAGENET_STD, overlap_prologue=not args.no_overlap,
                                  prefetch_next=pf)
        odt = torch.bfloat16
    else:
        aug = [None] * (Wu + K)
        params = st.decode_params(H, Wd, dtype=torch.float32, precision=precision,
                                  overlap_prologue=not args.no_overlap, prefetch_next=pf)
        odt = torch.float32
    out = torch.empty((B, 3, H, Wd), dtype=odt, device="cuda")

    def step(k):
        st.decode(ids[k], out=out, aug=aug[k], params=params, check=False, next_ids=ids[k + 1] if pf else None)

    for k in range(Wu):
        step(k)
    torch.cuda.synchronize()
    # capture exactly K decode launches in one CUDA graph (on a warmed side stream)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(Wu)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for k in range(K):
            step(Wu + k)
    sampler = ClockSampler(local)
    sampler.start()
    # keep the GPU busy ~0.5 s right up to the timed replay (loaded clocks, no idle gap)
    t_end = time.perf_counter() + 0.5
    while time.perf_counter() < t_end:
        graph.replay()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
        graph.replay()  # re-warm after the barrier's host round trip
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with stage("timed"):
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
    elapsed = e0.elapsed_time(e1) * 1e-3
    # keep the same work running >= 1.5 s so the clock sampler sees the loaded state
    t_end = time.perf_counter() + max(0.0, 1.5 - elapsed)
    sustain = []
    while time.perf_counter() < t_end:
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        graph.replay()
        a1.record()
        torch.cuda.synchronize()
        sustain.append(a0.elapsed_time(a1) * 1e-3)
    clocks = sampler.stop()
    del graph
    elapsed_max = reduce_max(elapsed, dist, "cuda")
    value = world * B * K / elapsed_max

    e2e = None
    if with_e2e and not args.no_e2e:
        e2e = measure_e2e(torch, dist, st, cfg, precision, ids, aug, B, H, Wd, K, world)

    sines = B * H * Wd * HIDDEN_SUM[cfg]
    dims = W["arch"]
    hid_flops = 2.0 * H * Wd * sum(dims[i] * dims[i + 1] for i in range(1, len(dims) - 2)) * B
    tensor_mult = 3 if precision == "fp32" else (1 if precision == "bf16" else 0)
    mufu_peak = peaks.get("mufu_sin_per_s")
    achieved = sines * K / elapsed
    meas = load_peaks()
    res = {
        "value": value, "unit": "images/s", "ms_per_step": 1e3 * elapsed_max / K, "steps": K, "warmup": Wu,
        "precision": precision,
        "dtype": "f32" if precision == "exact" else "bf16x3" if precision == "fp32" else "bf16",
        "config": {"workload": W["desc"], "precision": precision, "batch_per_gpu": B, "out": f"{H}x{Wd}",
                   "store_records_per_gpu": len(st), "store_records_total": int(st.info.total_records),
                   "store_bytes_per_gpu": int(st.info.device_bytes),
                   "l2": "inputs larger than L2: each step decodes a fresh random batch from a store > 126 MB"
                   if st.info.device_bytes > 126e6 else "store smaller than L2",
                   "parallelism": f"image-sharded x{world} (Store shard k % {world}), no decode collective",
                   "timing": "CUDA graph of K launches", "prologue_overlap": not args.no_overlap,
                   "next_batch_prefetch": "step k passes step k+1's ids; the narrow-net kernel prefetches their "
                   "record slots into L2 after its phase 1" if not args.no_prefetch else None,
                   "store_build_s": round(build_s, 2),
                   "store_source": "GPU generator (synth.gpu_store_bytes) -> .rinr bytes -> Store"},
        "roofline": {"bound": "mufu", "achieved": achieved / 1e9, "peak": mufu_peak / 1e9 if mufu_peak else None,
                     "unit": "Gsin/s", "frac": achieved / mufu_peak if mufu_peak else None,
                     "traffic": load_traffic(cfg, precision),
                     "per_launch": {"sines": sines, "hidden_tensor_flops": hid_flops * max(tensor_mult, 1),
                                    "algorithmic_sines_per_image": H * Wd * HIDDEN_SUM[cfg]},
                     "peak_source": "measured in this run by a MUFU.SIN microbenchmark (rinr_diag_launch)",
                     "tensor_frac_of_measured_bf16": (hid_flops * tensor_mult * K / elapsed) /
                     (meas.get("bf16_tflops", 1652.1) * 1e12) if tensor_mult else 0.0},
        "gpu_launches": K,
        "clocks": clocks,
        "sustain_ms_per_step": 1e3 * float(np.median(sustain)) / K if sustain else None,
    }
    if e2e:
        res["e2e"] = e2e
    if own:
        st.close()
    return res


def measure_e2e(torch, dist, st, cfg, precision, ids, aug, B, H, Wd, K, world):
    """Public API with host buffers: pinned ids in, NHWC f32 ImageBuffer batch out."""
    from paper_2306_16699_b200.store import IMAGENET_MEAN, IMAGENET_STD
    from paper_2306_16699_b200.trace import stage
    E = min(K, 50)
    ids_host = ids[:E].cpu().pin_memory()
    p_e2e = st.decode_params(H, Wd, dtype=torch.float32, layout="nhwc", precision=precision,
                             aug_mode="crop" if cfg == "c3" else None,
                             mean=IMAGENET_MEAN if cfg == "c3" else None,
                             std=IMAGENET_STD if cfg == "c3" else None)
    aug_host = [a.cpu().pin_memory() if a is not None else None for a in aug[:E]]
    # double-buffered device output; each step's D2H runs on two copy streams
    # (halves of the batch, two DMA engines) while the next step's H2D +
    # decode proceed on the main stream
    out_dev = [torch.empty((B, H, Wd, 3), dtype=torch.float32, device="cuda") for _ in range(2)]
    out_host = [torch.empty((B, H, Wd, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
    ids_dev = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
    aug_dev = [torch.empty((B, 5), dtype=torch.float32, device="cuda") for _ in range(2)]
    cstreams = [torch.cuda.Stream(), torch.cuda.Stream()]
    dec_done = [torch.cuda.Event() for _ in range(2)]
    copy_done = [[torch.cuda.Event() for _ in range(2)] for _ in range(2)]
    for sl in range(2):
        for c in range(2):
            copy_done[sl][c].record()
    half = B // 2
    main = torch.cuda.current_stream()

    def e2e_step(k):
        sl = k % 2
        for c in range(2):
            main.wait_event(copy_done[sl][c])  # out_dev[sl] / out_host[sl] free again
        ids_dev[sl].copy_(ids_host[k], non_blocking=True)
        a = None
        if aug_host[k] is not None:
            aug_dev[sl].copy_(aug_host[k], non_blocking=True)
            a = aug_dev[sl]
        st.decode(ids_dev[sl], out=out_dev[sl], aug=a, params=p_e2e, check=False)
        dec_done[sl].record(main)
        for c, (lo, hi) in enumerate(((0, half), (half, B))):
            with torch.cuda.stream(cstreams[c]):
                cstreams[c].wait_event(dec_done[sl])
                out_host[sl][lo:hi].copy_(out_dev[sl][lo:hi], non_blocking=True)
                copy_done[sl][c].record(cstreams[c])

    for k in range(min(3, E)):
        e2e_step(k)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with stage("e2e"):
        q0.record()
        for k in range(E):
            e2e_step(k)
        for sl in range(2):  # the region ends when the last results are on the host
            for c in range(2):
                main.wait_event(copy_done[sl][c])
        q1.record()
        torch.cuda.synchronize()
    et = reduce_max(q0.elapsed_time(q1) * 1e-3, dist, "cuda")
    return {"value": world * B * E / et, "unit": "images/s",
            "h2d_bytes_per_step": B * 8 + (B * 20 if cfg == "c3" else 0),
            "d2h_bytes_per_step": B * H * Wd * 3 * 4, "steps": E,
            "path": "Store.decode (C ABI rinr_decode) with pinned host ids in / NHWC f32 ImageBuffer batch out; "
                    "D2H of step k on two copy streams overlaps step k+1's H2D + decode"}


def measure_dropin(torch, n: int = 1024, reps: int = 3) -> dict:
    """The reference-API drop-in: rinr.decode_batch(models, 32, 32) on host
    InrModels of config c2 (decoder.py:39-61), wall-clock per call."""
    from paper_2306_16699_b200 import decode_batch, synth
    mb = synth.config2(n, seed=7, exact=False)
    models = [mb.model(i) for i in range(n)]
    decode_batch(models[:64], 32, 32)  # warm: library, allocator
    times = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        imgs = decode_batch(models, 32, 32)
        times.append(time.perf_counter() - t0)
    assert len(imgs) == n and imgs[0].pixels.shape == (32, 32, 3)
    t = float(np.median(times))
    return {"value": n / t, "unit": "images/s", "models_per_call": n, "ms_per_call": 1e3 * t,
            "path": "paper_2306_16699_b200.decode_batch (what install() binds to rinr.decode_batch): validate, "
                    "group, serialise (vectorised writer), transient Store, one fused decode, ImageBuffers; "
                    "host InrModels in, host ImageBuffers out, wall clock"}


def dist_env():
    """(rank, world, local GPU, backend).  RINR_BENCH_BACKEND=gloo with
    RINR_BENCH_ONE_GPU=1 runs every rank on cuda:0 (the multi-rank test of
    this script on a one-GPU box, tests/test_gpu_bench_multirank.py); real
    runs use NCCL, one process per GPU."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if os.environ.get("RINR_BENCH_ONE_GPU") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local, os.environ.get("RINR_BENCH_BACKEND", "nccl")


def init_dist(torch, world, local, backend):
    if world <= 1:
        return None
    import torch.distributed as dist
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return dist


def run_ours(args):
    rank, world, local, backend = dist_env()
    head = args.config
    subs = [] if (args.no_subs or head != "c2") else ["c1", "c3"]
    precision = args.precision or "fp32"

    # CPU baselines first (fork-based pool before CUDA is initialised), rank 0 at N=1 only
    cpu = {}
    if rank == 0 and world == 1 and not args.no_cpu:
        for cfg in [head] + subs:
            ips, sample, cores, _ = cpu_measure(cfg, workload(cfg))
            cpu[cfg] = {"value": ips, "unit": "images/s", "cores": cores, "kind": "port", "sample": sample}

    import torch
    torch.cuda.set_device(local)
    dist = init_dist(torch, world, local, backend)
    from paper_2306_16699_b200 import _native

    lib = _native.lib()
    peaks = measure_peaks(torch, lib)
    res = {head: measure_decode(torch, dist, head, precision, args, rank, world, local, peaks)}
    dropin = measure_dropin(torch) if (head == "c2" and rank == 0 and not args.no_e2e) else None
    for cfg in subs:
        if cfg == "c3":
            W = workload(cfg)
            st, build_s = open_store(torch, cfg, W, W["records"], rank, world, local)
            r = measure_decode(torch, dist, cfg, "fp32", args, rank, world, local, peaks, st, build_s)
            rb = measure_decode(torch, dist, cfg, "bf16", args, rank, world, local, peaks, st, build_s,
                                with_e2e=False)
            st.close()
            r["bf16"] = {k: rb[k] for k in ("value", "ms_per_step", "roofline", "clocks", "dtype")}
            r["bf16"]["parity"] = "per-image PSNR vs the reference decode >= 48 dB (10-layer nets, tests/conftest.py)"
            res[cfg] = r
        else:
            res[cfg] = measure_decode(torch, dist, cfg, precision, args, rank, world, local, peaks)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0

    h = res[head]
    line = {
        "metric": "decoded images/sec", "value": h["value"], "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": h["dtype"], "data": "synthetic",
        "config": h["config"], "roofline": h["roofline"], "gpu_launches": h["gpu_launches"],
        "clocks": h["clocks"], "sustain_ms_per_step": h["sustain_ms_per_step"],
    }
    line["roofline"]["measured_pipe_peaks"] = peaks
    if "e2e" in h:
        line["e2e"] = h["e2e"]
    if dropin:
        line["e2e_dropin"] = dropin
    if head in cpu:
        line["cpu_baseline"] = cpu[head]
    for cfg in subs:
        sub = res[cfg]
        if cfg in cpu:
            sub["cpu_baseline"] = cpu[cfg]
        line[cfg] = sub
        line["gpu_launches"] += sub["gpu_launches"] + sub.get("bf16", {}).get("gpu_launches", 0)
    print(json.dumps(line), flush=True)
    return 0


def run_train(args):
    """C4 / C5: end-to-end ResNet-18 training fed by the fused decode."""
    import torch
    import torchvision
    W = workload(args.config)
    rank, world, local, backend = dist_env()
    torch.cuda.set_device(local)
    dist = init_dist(torch, world, local, backend)
    from paper_2306_16699_b200 import train
    # c5: one 1M-record archive sharded over the ranks; c4: 16,384 records per GPU
    # (--store-records: records per GPU)
    total = args.store_records * world if args.store_records else (
        W["records"] if args.config == "c5" else W["records"] * world)
    t0 = time.perf_counter()
    st = train.open_sharded_store(W["synth"], total, rank, world, device=f"cuda:{local}", seed=4242)
    build_s = time.perf_counter() - t0
    precision = args.precision or "bf16"
    loop = train.DecodeTrainLoop(st, W["h"], W["w"], W["batch"], W["classes"], precision=precision,
                                 aug="crop" if W["h"] == 224 else "offset", seed=rank,
                                 ddp=dist is not None, device=f"cuda:{local}")
    K, Wu = args.steps, args.warmup
    for _ in range(Wu):
        loop.step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    t_end = time.perf_counter() + 0.3
    while time.perf_counter() < t_end:
        loop.step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        loss = loop.step()
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    elapsed = reduce_max(e0.elapsed_time(e1) * 1e-3, dist, "cuda")
    value = world * W["batch"] * K / elapsed
    dec_s = reduce_max(loop.time_decode_only(K), dist, "cuda")
    static_s = reduce_max(loop.time_train_only(K), dist, "cuda")
    final_loss = float(loss.item())
    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": "decoded+trained images/sec", "value": value, "unit": "images/s", "n_gpus": world, "steps": K,
        "warmup": Wu, "ms_per_step": 1e3 * elapsed / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": W["desc"], "batch_per_gpu": W["batch"], "store_records_per_gpu": len(st),
                   "store_records_total": int(st.info.total_records), "precision": precision,
                   "parallelism": f"DDP x{world} (NCCL gradient all-reduce), Store shard k % {world}" if world > 1
                   else "single GPU", "store_build_s": round(build_s, 2)},
        "decode_ms_per_step": 1e3 * dec_s / K,
        "decode_share_of_step": dec_s / elapsed,
        "static_batch_images_per_s": world * W["batch"] * K / static_s,
        "final_loss": final_loss,
        "gpu_launches": K,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    args = parse_args(argv)
    if args.config in ("c4", "c5"):
        if args.impl == "reference":
            rank = int(os.environ.get("RANK", "0"))
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "the reference has no GPU training path "
                                  "(SPEC.md:8 puts ResNet-18 training out of scope)"}), flush=True)
            return 0
        return run_train(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
