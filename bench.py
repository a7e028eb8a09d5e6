#!/usr/bin/env python
"""Decode throughput bench (BASELINE.json metric: decoded images/sec).

Workload (N=1 line = BASELINE config 2, the config the metric is quoted on):
  c2: batch of 1024 records, 32x32 output, arch [2,15,15,3], each record
      R1-initialised, L1-pruned to a per-record dynamic ratio (mean ~15%) and
      affine8-quantised, held in an HBM store of --store-records records per
      GPU (default 262,144 ~ 190 MB > 126 MB L2; each step samples a fresh
      random batch of ids from it, so the records it reads are not L2-resident).
  c3: batch of 256 records of arch [2,40x9,3] at 224x224 with random-resized-
      crop + flip + ImageNet normalise, bf16 NCHW out (--config c3).
A step = one fused decode launch over one batch (dequant prologue + MLP +
epilogue).  `value` is device throughput with ids resident in HBM, timed with
CUDA events around a CUDA-graph replay of exactly --steps launches, max over
ranks.  `e2e` runs the same steps through the public API with host buffers:
per step H2D of the ids from pinned memory, decode, D2H of the decoded
ImageBuffer-layout (NHWC f32) batch into pinned memory.

`--impl reference` times the reference algorithm on the host CPU instead
(the numpy oracle port of rinr.decode_batch, oracle/rinr_oracle.py — the
reference package itself cannot travel to the GPU box), with one worker
process per core, over the same config and batch.

Multi-GPU (torchrun): each rank holds its own shard of the store and decodes
its own batch; there is no collective in the decode (scaling "weak").
"""

from __future__ import annotations

import argparse
import json
import math
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
    ap.add_argument("--store-records", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="do not let a decode's prologue overlap the previous decode (PDL off)")
    return ap.parse_args(argv)


def workload(cfg: str):
    if cfg in ("c4", "c5"):
        return dict(batch=64, h=224, w=224, arch=[2] + [40] * 9 + [3], records=4096, desc=(
            f"{cfg}: ResNet-18 training step (SGD lr 1e-2, wd 5e-4, bf16 autocast, channels_last; PAPER.md:446) "
            "fed by on-the-fly decode of 64 affine8+25%-pruned [2,40x9,3] records per GPU at 224x224 with "
            "random-resized-crop+flip+ImageNet normalise (bf16 NCHW)" +
            (", DDP over NCCL, store sharded by record" if cfg == "c5" else "")))
    if cfg == "c1":
        return dict(batch=256, h=32, w=32, arch=[2, 15, 15, 3], records=262144, desc=(
            "c1: fp32 dense [2,15,15,3] random-init (R1) records, batch 256, 32x32, fp32 NCHW out"))
    if cfg == "c2":
        return dict(batch=1024, h=32, w=32, arch=[2, 15, 15, 3], records=262144, desc=(
            "c2: quantised(affine8)+pruned(mean~15%) [2,15,15,3] records, batch 1024, 32x32, fp32 NCHW out"))
    return dict(batch=256, h=224, w=224, arch=[2] + [40] * 9 + [3], records=4096, desc=(
        "c3: affine8 + 25%-pruned [2,40x9,3] records, batch 256, 224x224, random-resized-crop+flip+ImageNet "
        "normalise, bf16 NCHW out"))


def store_bytes(cfg: str, n: int, seed: int) -> bytes:
    from paper_2306_16699_b200 import synth
    if cfg == "c1":
        mb = synth.tweak_r1(synth.random_batch(synth.ARCH_A, n, seed))
        return synth.archive_bytes(mb)
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
    data = store_bytes(cfg, n_rec, seed=12345)
    pool = CpuPool(data, W["h"], W["w"], cores)
    rng = np.random.default_rng(0)
    B = W["batch"]
    try:
        # calibrate: one warm batch
        ids = rng.integers(0, n_rec, B if cfg != "c3" else cores)
        aug = crop_params_np(len(ids), 0) if cfg == "c3" else None
        t = pool.run(ids, aug)
        per_img = t / len(ids)
        times = []
        if steps is None:  # bounded sample: ~10-30 s of CPU work across the cores
            n = min(262144, cores * 8192) if cfg != "c3" else cores * 8
            ids = rng.integers(0, n_rec, n)
            aug = crop_params_np(n, 1) if cfg == "c3" else None
            t = pool.run(ids, aug)
            sample = (f"{n} images of {cfg} ({W['h']}x{W['w']}) decoded by the oracle port of rinr.decode_batch "
                      f"(net.forward + clip{'+ crop/normalise' if cfg == 'c3' else ''}) from pre-materialised "
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


def run_reference(args, W):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    total = args.warmup + args.steps
    _, sample, cores, times = cpu_measure(args.config, W, steps=total)
    t = sum(times[args.warmup:])
    per_step = W["batch"] if args.config != "c3" else max(cores, 16)
    value = per_step * args.steps / t
    line = {
        "impl": "reference", "metric": "decoded images/sec", "value": value, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": W["desc"], "cpu": cpu_model()},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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


def load_traffic(cfg):
    try:
        d = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
        return d.get(cfg, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def run_ours(args, W):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = args.config
    precision = args.precision or ("bf16" if cfg == "c3" else "fp32")

    # CPU baseline first (fork-based pool before CUDA is initialised).
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ips, sample, cores, _ = cpu_measure(cfg, W)
        cpu = {"value": ips, "unit": "images/s", "cores": cores, "kind": "port", "sample": sample}

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2306_16699_b200 import Store, _native
    from paper_2306_16699_b200.store import IMAGENET_MEAN, IMAGENET_STD, resized_crop_params

    lib = _native.lib()
    R = args.store_records or W["records"]
    t0 = time.perf_counter()
    data = store_bytes(cfg, R, seed=1000 * rank)
    st = Store(data, device=f"cuda:{local}")
    build_s = time.perf_counter() - t0
    del data
    B, H, Wd = W["batch"], W["h"], W["w"]
    K, Wu = args.steps, args.warmup
    gen = torch.Generator(device="cuda").manual_seed(rank)
    ids = torch.randint(0, len(st), (Wu + K, B), device="cuda", generator=gen, dtype=torch.int64)
    if cfg == "c3":
        aug = [resized_crop_params(B, generator=torch.Generator().manual_seed(1000 * rank + s)).cuda()
               for s in range(Wu + K)]
        params = st.decode_params(H, Wd, dtype=torch.bfloat16, precision=precision, aug_mode="crop",
                                  mean=IMAGENET_MEAN, std=IMAGENET_STD, overlap_prologue=not args.no_overlap)
        odt = torch.bfloat16
    else:
        aug = [None] * (Wu + K)
        params = st.decode_params(H, Wd, dtype=torch.float32, precision=precision,
                                  overlap_prologue=not args.no_overlap)
        odt = torch.float32
    out = torch.empty((B, 3, H, Wd), dtype=odt, device="cuda")

    def step(k):
        st.decode(ids[k], out=out, aug=aug[k], params=params, check=False)

    # warm-up: W steps plus ~0.5 s so clocks reach their loaded state
    for k in range(Wu):
        step(k)
    torch.cuda.synchronize()
    t_end = time.perf_counter() + 0.5
    while time.perf_counter() < t_end:
        for k in range(Wu):
            step(k)
        torch.cuda.synchronize()

    # capture exactly K decode launches in one CUDA graph
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(Wu)  # stream-side warm launch
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):  # the stream warmed above (its decode workspaces exist)
        for k in range(K):
            step(Wu + k)
    graph.replay()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.25)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
    elapsed_max = reduce_max(elapsed, dist, "cuda")
    value = world * B * K / elapsed_max

    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        E = min(K, 50)
        ids_host = ids[:E].cpu().pin_memory()
        p_e2e = st.decode_params(H, Wd, dtype=torch.float32, layout="nhwc", precision=precision,
                                 aug_mode="crop" if cfg == "c3" else None,
                                 mean=IMAGENET_MEAN if cfg == "c3" else None,
                                 std=IMAGENET_STD if cfg == "c3" else None)
        aug_host = [a.cpu().pin_memory() if a is not None else None for a in aug[:E]]
        # double-buffered device output; each step's D2H runs on two copy
        # streams (halves of the batch, two DMA engines) while the next step's
        # H2D + decode proceed on the main stream
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
        q0.record()
        for k in range(E):
            e2e_step(k)
        for sl in range(2):  # the region ends when the last results are on the host
            for c in range(2):
                main.wait_event(copy_done[sl][c])
        q1.record()
        torch.cuda.synchronize()
        et = q0.elapsed_time(q1) * 1e-3
        et = reduce_max(et, dist, "cuda")
        e2e = {"value": world * B * E / et, "unit": "images/s", "h2d_bytes_per_step": B * 8 + (B * 20 if cfg == "c3"
                                                                                           else 0),
               "d2h_bytes_per_step": B * H * Wd * 3 * 4, "steps": E,
               "path": "Store.decode (C ABI rinr_decode) with pinned host ids in / NHWC f32 ImageBuffer batch out; "
                       "D2H of step k on two copy streams overlaps step k+1's H2D + decode"}

    peaks_meas = measure_peaks(torch, lib) if rank == 0 else {}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0

    sines = B * H * Wd * HIDDEN_SUM[cfg]
    achieved = sines * K / elapsed
    mufu_peak = peaks_meas.get("mufu_sin_per_s")
    dims = W["arch"]
    hid_flops = 2.0 * H * Wd * sum(dims[i] * dims[i + 1] for i in range(1, len(dims) - 2)) * B
    tensor_mult = 3 if precision == "fp32" else (1 if precision == "bf16" else 0)
    peaks = load_peaks()
    line = {
        "metric": "decoded images/sec", "value": value, "unit": "images/s", "n_gpus": world, "steps": K,
        "warmup": Wu, "ms_per_step": 1e3 * elapsed_max / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if precision == "exact" else "bf16x3" if precision == "fp32" else "bf16",
        "data": "synthetic",
        "config": {"workload": W["desc"], "precision": precision, "batch_per_gpu": B, "out": f"{H}x{Wd}",
                   "store_records_per_gpu": R, "store_bytes_per_gpu": int(st.info.device_bytes),
                   "l2": "inputs larger than L2: each step decodes a fresh random batch from a store > 126 MB"
                   if st.info.device_bytes > 126e6 else "store smaller than L2",
                   "parallelism": f"image-sharded x{world}, no decode collective", "timing": "CUDA graph of K launches",
                   "prologue_overlap": not args.no_overlap,
                   "store_build_s": round(build_s, 2)},
        "roofline": {"bound": "mufu", "achieved": achieved / 1e9, "peak": mufu_peak / 1e9 if mufu_peak else None,
                     "unit": "Gsin/s", "frac": achieved / mufu_peak if mufu_peak else None,
                     "traffic": load_traffic(cfg),
                     "per_launch": {"sines": sines, "hidden_tensor_flops": hid_flops * max(tensor_mult, 1)},
                     "peak_source": "measured in this run by a MUFU.SIN microbenchmark (rinr_diag_launch)",
                     "tensor_frac_of_measured_bf16": (hid_flops * tensor_mult * K / elapsed) /
                     (peaks.get("bf16_tflops", 1669.7) * 1e12) if tensor_mult else 0.0,
                     "measured_pipe_peaks": peaks_meas},
        "gpu_launches": K,
        "clocks": clocks,
        "sustain_ms_per_step": 1e3 * float(np.median(sustain)) / K if sustain else None,
    }
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    st.close()
    return 0


def run_train(args, W):
    """C4 / C5: end-to-end ResNet-18 training fed by the fused decode."""
    import torch
    import torchvision
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2306_16699_b200 import Store
    from paper_2306_16699_b200.store import IMAGENET_MEAN, IMAGENET_STD, resized_crop_params

    R = args.store_records or W["records"]
    t0 = time.perf_counter()
    # every rank holds its own shard: records k with k % world == rank of a world*R store
    st = Store(store_bytes("c3", R, seed=1000 * rank), device=f"cuda:{local}")
    build_s = time.perf_counter() - t0
    B, H, Wd = W["batch"], W["h"], W["w"]
    K, Wu = args.steps, args.warmup
    precision = args.precision or "bf16"
    params = st.decode_params(H, Wd, dtype=torch.bfloat16, precision=precision, aug_mode="crop",
                              mean=IMAGENET_MEAN, std=IMAGENET_STD)
    model = torchvision.models.resnet18(num_classes=100).cuda().to(memory_format=torch.channels_last)
    if dist:
        model = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
    opt = torch.optim.SGD(model.parameters(), lr=1e-2, momentum=0.9, weight_decay=5e-4)
    lossf = torch.nn.CrossEntropyLoss()
    gen = torch.Generator(device="cuda").manual_seed(rank)
    ids = torch.randint(0, len(st), (Wu + K, B), device="cuda", generator=gen)
    labels = torch.randint(0, 100, (Wu + K, B), device="cuda", generator=gen)
    aug = torch.stack([resized_crop_params(B, generator=torch.Generator().manual_seed(1000 * rank + s))
                       for s in range(Wu + K)]).cuda()
    xbuf = torch.empty((B, 3, H, Wd), dtype=torch.bfloat16, device="cuda").to(memory_format=torch.contiguous_format)

    def train_step(x, y):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = lossf(model(x.contiguous(memory_format=torch.channels_last)), y)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        return loss

    def step(k, decode=True):
        if decode:
            st.decode(ids[k], out=xbuf, aug=aug[k], params=params, check=False)
        return train_step(xbuf, labels[k])

    def timed(n0, n, decode=True):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(n0, n0 + n):
            loss = step(k, decode)
        e1.record()
        torch.cuda.synchronize()
        return reduce_max(e0.elapsed_time(e1) * 1e-3, dist, "cuda"), float(loss.item())

    for k in range(Wu):
        step(k)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    elapsed, loss = timed(Wu, K)
    clocks = sampler.stop()
    value = world * B * K / elapsed
    # decode alone (same launches) and the training step on a static pre-decoded batch
    torch.cuda.synchronize()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record()
    for k in range(Wu, Wu + K):
        st.decode(ids[k], out=xbuf, aug=aug[k], params=params, check=False)
    d1.record()
    torch.cuda.synchronize()
    dec_s = d0.elapsed_time(d1) * 1e-3
    static_s, _ = timed(Wu, K, decode=False)
    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": "decoded+trained images/sec", "value": value, "unit": "images/s", "n_gpus": world, "steps": K,
        "warmup": Wu, "ms_per_step": 1e3 * elapsed / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": W["desc"], "batch_per_gpu": B, "store_records_per_gpu": R, "precision": precision,
                   "parallelism": f"DDP x{world} (NCCL gradient all-reduce), image-sharded store" if world > 1
                   else "single GPU", "store_build_s": round(build_s, 2)},
        "decode_ms_per_step": 1e3 * dec_s / K,
        "decode_share_of_step": dec_s / elapsed,
        "static_batch_images_per_s": world * B * K / static_s,
        "final_loss": loss,
        "gpu_launches": K,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    args = parse_args(argv)
    W = workload(args.config)
    if args.config in ("c4", "c5"):
        if args.impl == "reference":
            rank = int(os.environ.get("RANK", "0"))
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "the reference has no GPU training path "
                                  "(SPEC.md:8 puts ResNet-18 training out of scope)"}), flush=True)
            return 0
        return run_train(args, W)
    if args.impl == "reference":
        return run_reference(args, W)
    return run_ours(args, W)


if __name__ == "__main__":
    sys.exit(main())
