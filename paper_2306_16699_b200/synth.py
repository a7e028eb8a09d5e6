"""Seeded synthetic INR stores for the BASELINE configs.

  C1  arch A [2,15,15,3], fp32 dense, seeds 0..n-1 with the reference's
      net.init draws (R0 literal, or R1: last layer w x 20, b = 0.5).
  C2  arch A, R1, per-record prune ratio dynamic_ratio(cifar, U(28, 37) dB)
      (mean ~15%), then affine8.
  C3  arch C [2,40x9,3], R1, 25% prune, affine8; decoded at 224 x 224.
Large stores (bench: inputs bigger than L2) use one vectorised generator
instead of per-record seeds; records are still written by the same writer.
"""

from __future__ import annotations

import numpy as np

from . import net
from .archive import serialize_batch
from .compressor import SCHEDULES, ModelBatch, dynamic_ratio_cifar, prune_l1_batch, quantize_batch
from .net import Architecture

ARCH_A = Architecture((2, 15, 15, 3))
ARCH_B = Architecture((2, *([32] * 9), 3))
ARCH_C = Architecture((2, *([40] * 9), 3))


def record_ids(n: int, start: int = 0) -> list:
    return [f"img{i:08d}" for i in range(start, start + n)]


def seeded_batch(arch: Architecture, seeds, source=(32, 32)) -> ModelBatch:
    """Per-record net.init(arch, seed) — the reference's exact draws."""
    mb = ModelBatch.from_models([net.init(arch, int(s)) for s in seeds])
    mb.source_h, mb.source_w = source
    return mb


def random_batch(arch: Architecture, n: int, seed: int, source=(32, 32)) -> ModelBatch:
    """Same distributions as net.init, one PCG64 stream for the whole batch."""
    rng = np.random.default_rng(seed)
    w, b, m = [], [], []
    for li, (fi, fo) in enumerate(zip(arch.dims[:-1], arch.dims[1:])):
        bound = 1.0 / fi if li == 0 else np.sqrt(6.0 / fi) / arch.omega
        w.append(rng.uniform(-bound, bound, size=(n, fo, fi)).astype(np.float32))
        b.append(np.zeros((n, fo), np.float32))
        m.append(np.ones((n, fo, fi), bool))
    return ModelBatch(arch, w, b, m, source[0], source[1])


def tweak_r1(mb: ModelBatch) -> ModelBatch:
    """R1: last layer w x 20 and bias 0.5 so outputs span both clamps."""
    mb.w[-1] = (mb.w[-1] * np.float32(20.0)).astype(np.float32)
    mb.b[-1] = np.full_like(mb.b[-1], 0.5)
    return mb


def cifar_ratios(n: int, seed: int) -> np.ndarray:
    """Per-record prune ratios dynamic_ratio(cifar, U(28, 37) dB), vectorised
    with the same IEEE operations as compressor.dynamic_ratio."""
    rng = np.random.default_rng(seed + 7919)
    p = rng.uniform(28.0, 37.0, n)
    sched = SCHEDULES["cifar"]
    out = np.where(p < sched.pieces[0][0], sched.below, sched.above)
    done = np.zeros(n, bool)
    for lo, hi, slope, intercept in sched.pieces:
        done |= p < lo  # the reference loop breaks here
        hit = ~done & (p <= hi)
        out = np.where(hit, slope * p + intercept, out)
        done |= hit
    return out


def config1(n: int = 256, variant: str = "R1") -> ModelBatch:
    mb = seeded_batch(ARCH_A, range(n))
    return tweak_r1(mb) if variant == "R1" else mb


def config2(n: int = 1024, seed: int = 0, exact: bool = True) -> ModelBatch:
    mb = seeded_batch(ARCH_A, range(seed, seed + n)) if exact else random_batch(ARCH_A, n, seed)
    mb = prune_l1_batch(tweak_r1(mb), cifar_ratios(n, seed))
    return quantize_batch(mb, "affine8")


def config3(n: int = 256, seed: int = 0, arch: Architecture = ARCH_C, exact: bool = True) -> ModelBatch:
    mb = seeded_batch(arch, range(seed, seed + n), (224, 224)) if exact else random_batch(arch, n, seed, (224, 224))
    mb = prune_l1_batch(tweak_r1(mb), 0.25)
    return quantize_batch(mb, "affine8")


def archive_bytes(mb: ModelBatch, start_id: int = 0) -> bytes:
    return serialize_batch(mb, record_ids(mb.n, start_id))


def gpu_store_bytes(config: str, n: int, seed: int = 0, device="cuda", chunk: int = 1 << 18) -> bytes:
    """Archive bytes of an n-record synthetic store of config 'c1', 'c2' or
    'c3', generated on the GPU: net.init's distributions from a seeded torch
    generator (R1 tweak), GPU prune_l1 to the config's ratios, GPU quantize
    and the GPU writer (transforms.serialize) — the same pipeline as the host
    generator, at GPU speed (a 1M-record c2 store in seconds)."""
    import torch  # noqa: PLC0415

    from . import transforms as T  # noqa: PLC0415
    arch = {"c1": ARCH_A, "c2": ARCH_A, "c3": ARCH_C}[config]
    src = (224, 224) if config == "c3" else (32, 32)
    gen = torch.Generator(device=device).manual_seed(seed)
    parts = []
    lens = []
    for s in range(0, n, chunk):
        k = min(chunk, n - s)
        ws, bs = [], []
        dims = arch.dims
        for li, (fi, fo) in enumerate(zip(dims[:-1], dims[1:])):
            bound = 1.0 / fi if li == 0 else float(np.sqrt(6.0 / fi) / arch.omega)
            ws.append(((torch.rand((k, fo * fi), generator=gen, device=device, dtype=torch.float64) * 2 - 1)
                       * bound).to(torch.float32))
            bs.append(torch.zeros((k, fo), device=device))
        ws[-1] = ws[-1] * np.float32(20.0)  # R1: last layer x 20, bias 0.5
        bs[-1] = torch.full_like(bs[-1], 0.5)
        dm = T.DeviceModels(arch, torch.cat(ws, 1).contiguous(), torch.ones((k, sum(w.shape[1] for w in ws)),
                            dtype=torch.uint8, device=device), torch.cat(bs, 1).contiguous(), src[0], src[1])
        q = None
        if config != "c1":
            ratio = torch.from_numpy(cifar_ratios(k, seed + s)) if config == "c2" else 0.25
            T.prune_l1(dm, ratio)
            q = T.quantize(dm, "affine8")
        buf = T.serialize(dm, q, id_prefix="img", first_id=s, id_width=8)
        cnt = int(np.frombuffer(buf[6:10].cpu().numpy().tobytes(), "<u4")[0])
        idx = buf[10:10 + 12 * cnt].cpu().numpy().view(np.dtype([("off", "<u8"), ("len", "<u4")]))
        parts.append(buf[10 + 12 * cnt:].cpu().numpy())
        lens.append(idx["len"].astype(np.int64))
    from .archive import _wrap  # noqa: PLC0415
    return _wrap(np.concatenate(parts), np.concatenate(lens))


def large_store_bytes(config: str, n: int, seed: int = 0, chunk: int = 65536) -> bytes:
    """A store of n records of config 'c2' or 'c3' built chunk by chunk (the
    bench uses stores larger than the 126 MB L2)."""
    from .archive import _wrap, _encode_batch_buffer  # noqa: PLC0415
    bufs, lens = [], []
    for s in range(0, n, chunk):
        k = min(chunk, n - s)
        if config == "c2":
            mb = config2(k, seed + s, exact=False)
        elif config == "c3":
            mb = config3(k, seed + s, exact=False)
        else:
            raise ValueError(config)
        buf, starts, body = _encode_batch_buffer(mb, record_ids(k, s))
        bufs.append(buf)
        lens.append(body + 4)
    return _wrap(np.concatenate(bufs), np.concatenate(lens))
