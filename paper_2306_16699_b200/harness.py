"""``bench``: the reference's decode-throughput harness (``rinr.bench.bench``,
bench.py:34-93) on the GPU path, with the same report type and fields.

Stages map onto the GPU pipeline:

  * ``load``: read the archive and ``rinr_store_create`` (host parse, CRC,
    one HBM upload);
  * ``dequantize``: ``rinr_dequantize`` of every record (CUDA events);
  * ``forward``: the fused decode kernel to u8 HWC, clamp and round half away
    included (CUDA events);
  * ``clamp_convert``: 0.0, because it is fused into ``forward``.

``digest`` is sha256 over the decoded 8-bit pixels in record order, like the
reference's.  It is deterministic from run to run and equals the reference
harness's digest on every golden store (tests/test_gpu_digest.py); in
general the GPU sums in a different order, so a value sitting exactly on a
u8 rounding boundary could land one level apart.  The throughput pass decodes all records in
batches of ``batch``.  ``jobs`` is validated, then ignored, because one launch
covers a batch.
"""

from __future__ import annotations

import hashlib
import time
from dataclasses import dataclass, field

import torch

from .errors import InvalidInputError
from .trace import stage


@dataclass
class BenchReport:
    """bench.py:21-31."""

    images: int
    pixels: int
    batch: int
    jobs: int
    stage_seconds: dict = field(default_factory=dict)
    wall_seconds: float = 0.0
    images_per_s: float = 0.0
    pixels_per_s: float = 0.0
    digest: str = ""


def bench(source, batch: int = 8, jobs: int = 1, out_h: int | None = None, out_w: int | None = None,
          device=None) -> BenchReport:
    """Measure decode performance of every record in an archive (path or bytes)."""
    from pathlib import Path

    from .store import Store
    if batch < 1 or jobs < 1:
        raise InvalidInputError("batch and jobs must be >= 1")
    stages = {"load": 0.0, "dequantize": 0.0, "forward": 0.0, "clamp_convert": 0.0}
    t0 = time.perf_counter()
    data = Path(source).read_bytes() if isinstance(source, (str, Path)) else source
    st = Store(data, device=device)
    torch.cuda.synchronize(st.device)
    stages["load"] = time.perf_counter() - t0
    try:
        n = len(st)
        ids = torch.arange(n, device=st.device)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        if n:  # first launch pays the lazy module load (~30 ms), not the stage
            st.dequantize(ids[:1])
        ev[0].record()
        st.dequantize(ids)
        ev[1].record()
        torch.cuda.synchronize(st.device)
        stages["dequantize"] = ev[0].elapsed_time(ev[1]) * 1e-3
        # group records by output size (native sizes may differ per record)
        sizes = {}
        for k in range(n):
            m = st.record_meta(k)
            hw = (out_h or m["source_h"], out_w or m["source_w"])
            sizes.setdefault(hw, []).append(k)
        hasher_parts = {}
        total_pixels = 0
        for (h, w), ks in sizes.items():
            kt = torch.tensor(ks, device=st.device)
            ev[0].record()
            u8 = st.decode(kt, h, w, dtype=torch.uint8, layout="nhwc", precision="exact", sin="accurate")
            ev[1].record()
            torch.cuda.synchronize(st.device)
            stages["forward"] += ev[0].elapsed_time(ev[1]) * 1e-3
            with stage("clamp_convert"):  # fused into forward; this range is the D2H of the u8 pixels
                host = u8.cpu().numpy()
            for k, img in zip(ks, host):
                hasher_parts[k] = img.tobytes()
            total_pixels += h * w * len(ks)
        hasher = hashlib.sha256()
        for k in range(n):
            hasher.update(hasher_parts[k])
        # throughput pass: batches of `batch` records, f32 decode as decode_batch returns
        torch.cuda.synchronize(st.device)
        t0 = time.perf_counter()
        with stage("throughput"):
            for (h, w), ks in sizes.items():
                for s in range(0, len(ks), batch):
                    st.decode(torch.tensor(ks[s:s + batch], device=st.device), h, w, layout="nhwc", check=False)
            torch.cuda.synchronize(st.device)
        wall = time.perf_counter() - t0
    finally:
        st.close()
    return BenchReport(images=n, pixels=total_pixels, batch=batch, jobs=jobs, stage_seconds=stages,
                       wall_seconds=wall, images_per_s=n / wall if wall > 0 else float("inf"),
                       pixels_per_s=total_pixels / wall if wall > 0 else float("inf"), digest=hasher.hexdigest())
