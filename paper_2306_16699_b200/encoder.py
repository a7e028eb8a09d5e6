"""Batched GPU encoder: the reference's per-image fit pipeline (``rinr.encoder``)
run for many images at once on the GPU.

The same three rounds, with the reference's names and arguments:

  * ``fit_round1``: overfit a fresh ``net.init`` model (encoder.py:100-113);
  * ``fit_full``: round 1, then round 2 (20% global magnitude prune + retrain)
    and round 3 (prune to the PSNR-scheduled total ratio + retrain)
    (encoder.py:116-146);
  * ``encode_dataset``: per-image seeds from ``derive_seed``, errors collected
    per image (encoder.py:147-235).

The ``*_batch`` variants take an [N, H, W, 3] f32 image tensor and fit all N
images with one kernel launch per round (``rinr_fit``, csrc/fit.cu: one CTA
per image, every Adam step of the round inside the launch).  Masking uses
the bit-exact GPU ``transforms.prune_l1``.  PSNR goes through the GPU render
+ ``transforms.psnr`` (the reference decodes with ``decoder.decode``).  The
trajectory is fp32 like the reference; the gradient summation order differs,
so results agree statistically (tests/test_gpu_encoder.py states the bars).
There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _native as N
from . import transforms as T
from .compressor import ModelBatch, dynamic_ratio, get_schedule
from .errors import ERR_STRUCTURAL, BatchItemError, InvalidInputError, StructuralError, TrainingError
from .image import ImageBuffer
from .net import Architecture, init

SIN_MODES = {"mufu": N.SIN_MUFU, "accurate": N.SIN_ACCURATE}


def cosine_lr(lr0: float, t: int, total: int) -> float:
    """Cosine decay from lr0 at t=0 to exactly 0 at t=total (encoder.py:28-30)."""
    return 0.5 * lr0 * (1.0 + math.cos(math.pi * t / total))


def derive_seed(global_seed: int, index: int) -> int:
    """Stable per-image seed: splitmix64 over (global seed, index) (encoder.py:146-152)."""
    mask = (1 << 64) - 1
    z = ((global_seed & mask) + (index + 1) * 0x9E3779B97F4A7C15) & mask
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
    return z ^ (z >> 31)


@dataclass(frozen=True)
class EncodeConfig:
    """encoder.py:33-52, plus ``sin`` (GPU sine unit: 'mufu' or 'accurate')."""

    arch: Architecture
    round1_lr: float = 5e-4
    round1_steps: int = 5000
    retrain_lr: float = 2e-4
    retrain_steps: int = 10000
    iterative_prune_ratio: float = 0.20
    skip_round2: bool = False
    schedule: str = "cifar"
    seed: int = 0
    sin: str = "mufu"

    def __post_init__(self):
        if self.round1_steps <= 0 or self.retrain_steps <= 0:
            raise InvalidInputError("step counts must be > 0")
        if self.round1_lr <= 0 or self.retrain_lr <= 0:
            raise InvalidInputError("learning rates must be > 0")
        if not (0.0 <= self.iterative_prune_ratio < 1.0):
            raise InvalidInputError("iterative_prune_ratio must be in [0, 1)")
        get_schedule(self.schedule)
        if self.sin not in SIN_MODES:
            raise InvalidInputError(f"sin must be one of {sorted(SIN_MODES)}")


@dataclass
class EncodeReport:
    """encoder.py:55-66."""

    psnr_after_round: list = field(default_factory=list)
    psnr_after_mask: list = field(default_factory=list)
    final_prune_ratio: float = 0.0
    loss_curve: list = field(default_factory=list)
    wall_time: float = 0.0


@dataclass
class DatasetReport:
    per_image: list = field(default_factory=list)
    failures: list = field(default_factory=list)

    @property
    def mean_psnr(self) -> float:
        vals = [r.psnr_after_round[-1] for r in self.per_image if r is not None]
        return float(np.mean(vals)) if vals else math.nan

    @property
    def mean_prune_ratio(self) -> float:
        vals = [r.final_prune_ratio for r in self.per_image if r is not None]
        return float(np.mean(vals)) if vals else math.nan


FitParams = N.FitParams


def _lib():
    return N.lib()


def _images(images, device) -> torch.Tensor:
    if isinstance(images, torch.Tensor):
        x = images
    else:
        x = torch.from_numpy(np.stack([im.as_float(np.float32) if isinstance(im, ImageBuffer) else
                                       np.asarray(im, np.float32) for im in images]))
    if x.dim() != 4 or x.shape[-1] != 3 or x.shape[0] < 1:
        raise InvalidInputError(f"images must be [N, H, W, 3], got {tuple(x.shape)}")
    return x.to(device=device, dtype=torch.float32).contiguous()


def init_batch(arch: Architecture, seeds, h: int, w: int, device="cuda") -> T.DeviceModels:
    """net.init per seed (the reference's PCG64 draws), uploaded."""
    mb = ModelBatch.from_models([init(arch, int(s)) for s in seeds])
    mb.source_h, mb.source_w = h, w
    return T.DeviceModels.from_batch(mb, device)


def _schedule(lr0: float, steps: int) -> np.ndarray:
    """[steps, 3] f32: the learning rate and Adam bias corrections of every
    step, computed exactly as encoder._train / net.Adam do (Python floats,
    cast to f32 where numpy's weak scalars meet the f32 arrays)."""
    t = np.arange(steps)
    lr = np.array([cosine_lr(lr0, int(i), steps) for i in t], np.float64)
    c1 = np.array([1.0 - 0.9 ** int(i + 1) for i in t], np.float64)
    c2 = np.array([1.0 - 0.999 ** int(i + 1) for i in t], np.float64)
    return np.stack([lr, c1, c2], 1).astype(np.float32)


def train_batch(dm: T.DeviceModels, images: torch.Tensor, lr0: float, steps: int, sin: str = "mufu"):
    """encoder._train for every model/image pair (in place).  Returns
    (curves [N, k] f64 numpy, status [N] int: 0 or failing step + 1)."""
    n, h, w = images.shape[0], images.shape[1], images.shape[2]
    stride = max(1, steps // 64)
    cap = (steps + stride - 1) // stride + 2
    curve = torch.empty((n, cap), dtype=torch.float64, device=images.device)
    status = torch.zeros(n, dtype=torch.int32, device=images.device)
    sched = torch.from_numpy(_schedule(lr0, steps)).to(images.device)
    p = FitParams(h, w, steps, SIN_MODES[sin], float(lr0), float(dm.arch.omega), cap, sched.data_ptr())
    dims, nl = T._dims(dm.arch)
    with torch.cuda.device(dm.w.device):  # launch on the tensors' device
        N.check(_lib().rinr_fit(dims, nl, n, dm.w.data_ptr(), dm.b.data_ptr(), dm.mask.data_ptr(), images.data_ptr(),
                                C.byref(p), curve.data_ptr(), status.data_ptr(), None, None, None,
                                T._stream(images.device)))
    return curve.cpu().numpy(), status.cpu().numpy()


def loss_and_grad_batch(dm: T.DeviceModels, images: torch.Tensor, sin: str = "mufu"):
    """net.loss_and_grad (net.py:217-265) for every model: (loss [N] f64,
    grad_w [N, P] f32 masked, grad_b [N, PB] f32); nothing is updated."""
    n, h, w = images.shape[0], images.shape[1], images.shape[2]
    gw = torch.empty_like(dm.w)
    gb = torch.empty_like(dm.b)
    loss = torch.empty(n, dtype=torch.float64, device=images.device)
    curve = torch.empty((n, 2), dtype=torch.float64, device=images.device)
    status = torch.zeros(n, dtype=torch.int32, device=images.device)
    p = FitParams(h, w, 0, SIN_MODES[sin], 0.0, float(dm.arch.omega), 2, None)
    dims, nl = T._dims(dm.arch)
    with torch.cuda.device(dm.w.device):  # launch on the tensors' device
        N.check(_lib().rinr_fit(dims, nl, n, dm.w.data_ptr(), dm.b.data_ptr(), dm.mask.data_ptr(), images.data_ptr(),
                                C.byref(p), curve.data_ptr(), status.data_ptr(), gw.data_ptr(), gb.data_ptr(),
                                loss.data_ptr(), T._stream(images.device)))
    return loss, gw, gb


def render(dm: T.DeviceModels, h: int, w: int, sin: str = "mufu") -> torch.Tensor:
    """Clipped [N, h, w, 3] decode of the models (decoder.decode)."""
    out = torch.empty((dm.n, h, w, 3), dtype=torch.float32, device=dm.w.device)
    dims, nl = T._dims(dm.arch)
    with torch.cuda.device(dm.w.device):  # launch on the tensors' device
        N.check(_lib().rinr_fit_render(dims, nl, dm.n, dm.w.data_ptr(), dm.b.data_ptr(), h, w, float(dm.arch.omega),
                                       SIN_MODES[sin], out.data_ptr(), T._stream(dm.w.device)))
    return out


def _psnr(dm, images, sin) -> np.ndarray:
    _, p = T.psnr(render(dm, images.shape[1], images.shape[2], sin), images)
    return p.cpu().numpy()


def _prune_ratio(dm: T.DeviceModels) -> np.ndarray:
    return 1.0 - dm.mask.sum(dim=1).cpu().numpy() / dm.mask.shape[1]


def _train_round(dm, images, lr0, steps, cfg, reports, alive, on_error):
    curves, status = train_batch(dm, images, lr0, steps, cfg.sin)
    for i in range(dm.n):
        if not alive[i]:
            continue
        if status[i]:
            err = TrainingError(f"loss became non-finite at step {status[i] - 1}", step=int(status[i] - 1))
            if on_error == "fail_fast":
                raise BatchItemError(i, err)
            alive[i] = err
            continue
        reports[i].loss_curve.extend(float(v) for v in curves[i] if not math.isnan(v))


def _prune_round(dm, ratios, alive, on_error):
    """Per-image prune (GPU prune_l1, check=False): an image whose prune would
    empty a layer fails alone, as it does in the reference's per-image loop
    (encoder.py:120-135); with fail_fast the first failure is raised."""
    status = T.prune_l1(dm, ratios, check=False).cpu().numpy()
    for i in np.nonzero(status)[0]:
        if not alive[i]:
            continue
        code = int(status[i])
        cause = (StructuralError if code == ERR_STRUCTURAL else InvalidInputError)(
            f"prune_l1 failed (status {code})")
        if on_error == "fail_fast":
            raise BatchItemError(int(i), cause)
        alive[i] = cause


def fit_round1_batch(images, cfg: EncodeConfig, seeds=None, device="cuda", on_error="fail_fast"):
    """Round 1 for every image: (DeviceModels, [EncodeReport])."""
    t0 = time.perf_counter()
    x = _images(images, device)
    n, h, w = x.shape[0], x.shape[1], x.shape[2]
    seeds = [cfg.seed] * n if seeds is None else list(seeds)
    dm = init_batch(cfg.arch, seeds, h, w, device)
    reports = [EncodeReport() for _ in range(n)]
    alive = [True] * n
    _train_round(dm, x, cfg.round1_lr, cfg.round1_steps, cfg, reports, alive, on_error)
    p = _psnr(dm, x, cfg.sin)
    ratio = _prune_ratio(dm)
    dt = (time.perf_counter() - t0) / n
    for i, r in enumerate(reports):
        r.psnr_after_round.append(float(p[i]))
        r.final_prune_ratio = float(ratio[i])
        r.wall_time = dt
    return dm, reports, alive


def fit_full_batch(images, cfg: EncodeConfig, seeds=None, device="cuda", on_error="fail_fast"):
    """The three-round pipeline for every image: (DeviceModels, [EncodeReport], alive)."""
    t0 = time.perf_counter()
    x = _images(images, device)
    dm, reports, alive = fit_round1_batch(x, cfg, seeds, device, on_error)
    psnr = np.array([r.psnr_after_round[0] for r in reports])
    if not cfg.skip_round2:
        _prune_round(dm, cfg.iterative_prune_ratio, alive, on_error)
        pm = _psnr(dm, x, cfg.sin)
        _train_round(dm, x, cfg.retrain_lr, cfg.retrain_steps, cfg, reports, alive, on_error)
        psnr = _psnr(dm, x, cfg.sin)
        for i, r in enumerate(reports):
            r.psnr_after_mask.append(float(pm[i]))
            r.psnr_after_round.append(float(psnr[i]))
    sched = get_schedule(cfg.schedule)
    ratios = np.array([dynamic_ratio(sched, float(v)) if not math.isnan(v) else 0.0 for v in psnr])
    _prune_round(dm, torch.from_numpy(ratios), alive, on_error)
    pm = _psnr(dm, x, cfg.sin)
    _train_round(dm, x, cfg.retrain_lr, cfg.retrain_steps, cfg, reports, alive, on_error)
    pf = _psnr(dm, x, cfg.sin)
    ratio = _prune_ratio(dm)
    dt = (time.perf_counter() - t0) / dm.n
    for i, r in enumerate(reports):
        r.psnr_after_mask.append(float(pm[i]))
        r.psnr_after_round.append(float(pf[i]))
        r.final_prune_ratio = float(ratio[i])
        r.wall_time = dt
    return dm, reports, alive


def _one(image: ImageBuffer, dm: T.DeviceModels):
    mb = dm.to_batch()
    mb.source_h, mb.source_w = image.h, image.w
    return mb.model(0)


def fit_round1(image: ImageBuffer, cfg: EncodeConfig):
    """encoder.fit_round1 (encoder.py:100-113) on the GPU: (InrModel, EncodeReport)."""
    dm, reports, _ = fit_round1_batch([image], cfg, [cfg.seed])
    return _one(image, dm), reports[0]


def fit_full(image: ImageBuffer, cfg: EncodeConfig):
    """encoder.fit_full (encoder.py:116-146) on the GPU: (InrModel, EncodeReport)."""
    dm, reports, _ = fit_full_batch([image], cfg, [cfg.seed])
    return _one(image, dm), reports[0]


def encode_dataset(images, cfg: EncodeConfig, parallelism: int = 1, ids=None, on_error: str = "fail_fast"):
    """encoder.encode_dataset (encoder.py:155-228): fit every image (all in one
    batch per round; ``parallelism`` is validated, then ignored) and collect
    the models into a DatasetArchive.  Images must share one size."""
    from .archive import ArchiveRecord, DatasetArchive
    if on_error not in ("fail_fast", "skip"):
        raise InvalidInputError(f"unknown on_error policy {on_error!r}")
    images = list(images) if not isinstance(images, torch.Tensor) else images
    if len(images) == 0:
        raise InvalidInputError("need at least one image")
    if parallelism < 1:
        raise InvalidInputError("parallelism must be >= 1")
    n = len(images)
    if ids is None:
        ids = [str(i) for i in range(n)]
    if len(ids) != n or len(set(ids)) != len(ids):
        raise InvalidInputError("ids must be unique and match the image count")
    seeds = [derive_seed(cfg.seed, i) for i in range(n)]
    dm, reports, alive = fit_full_batch(images, cfg, seeds, on_error=on_error)
    mb = dm.to_batch()
    report = DatasetReport()
    records = []
    for i in range(n):
        if alive[i] is not True:
            report.failures.append((i, str(alive[i])))
            continue
        records.append(ArchiveRecord(ids[i], mb.model(i)))
        report.per_image.append(reports[i])
    return DatasetArchive(records=records), report


__all__ = ["EncodeConfig", "EncodeReport", "DatasetReport", "cosine_lr", "derive_seed", "fit_round1", "fit_full",
           "fit_round1_batch", "fit_full_batch", "encode_dataset", "train_batch", "loss_and_grad_batch", "render",
           "init_batch"]
