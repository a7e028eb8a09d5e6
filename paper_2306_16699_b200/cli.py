"""Command line: ``decode`` and ``encode`` on the GPU.

Mirrors the reference CLI's subcommands of the same names (cli.py:107-176,
332-355): same arguments, JSON-lines output with ``--json``, and exit codes
0 ok / 1 usage / 2 data-format-integrity / 3 numeric.

  * ``decode``: the fused GPU decode writes u8 HWC directly (round half away
    from zero, image.py:49-55) for every requested record at its native size
    or ``--size``, one launch per output size; each image becomes a PNG via
    Pillow, as in the reference.
  * ``encode``: rasters -> GPU ``encode_dataset`` (all images of one size in
    one batch) -> ``.rinr`` archive.

    python -m paper_2306_16699_b200.cli decode data.rinr -o out_dir [--size HxW] [--ids a,b] [--json]
    python -m paper_2306_16699_b200.cli encode img_dir -o data.rinr [--round1-steps N ...] [--json]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

from .errors import BatchItemError, NumericError, RinrError

RASTER_SUFFIXES = {".png", ".bmp", ".jpg", ".jpeg", ".ppm", ".pgm", ".tif", ".tiff", ".webp"}


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (cli.py:29-34)
        self.print_usage(sys.stderr)
        self.exit(1, f"{self.prog}: error: {message}\n")


def _parse_size(text: str):
    try:
        h, w = (int(x) for x in text.lower().split("x"))
        return h, w
    except ValueError:
        raise argparse.ArgumentTypeError(f"--size expects HxW (e.g. 64x64), got {text!r}") from None


def _emit(args, record: dict, text: str) -> None:
    print(json.dumps(record) if args.json else text)


def _save_png(pixels_u8: np.ndarray, path) -> None:
    from PIL import Image
    Image.fromarray(pixels_u8, "RGB").save(path, format="PNG")


def decode_to_png(source, out_dir, size=None, ids=None, device=None):
    """Decode records of an archive (path or bytes) to PNGs; returns
    [(record id, path, h, w)] in archive order."""
    import torch

    from .store import Store
    with Store(source, device=device) as st:
        metas = [st.record_meta(k) for k in range(len(st))]
        want = None if ids is None else list(ids)
        if want is not None:
            have = {m["id"] for m in metas}
            missing = set(want) - have
            if missing:
                raise RinrError(f"ids not in archive: {sorted(missing)}")
            sel = [k for k, m in enumerate(metas) if m["id"] in set(want)]
        else:
            sel = list(range(len(metas)))
        out_dir = Path(out_dir)
        out_dir.mkdir(parents=True, exist_ok=True)
        groups = {}
        for k in sel:
            hw = size if size else (metas[k]["source_h"], metas[k]["source_w"])
            groups.setdefault(hw, []).append(k)
        done = {}
        for (h, w), ks in groups.items():
            pix = st.decode(torch.tensor(ks), h, w, dtype=torch.uint8, layout="nhwc", precision="exact",
                            sin="accurate").cpu().numpy()
            for k, img in zip(ks, pix):
                dest = out_dir / f"{metas[k]['id'].replace('/', '_')}.png"
                _save_png(img, dest)
                done[k] = (metas[k]["id"], dest, h, w)
        return [done[k] for k in sel]


def _cmd_decode(args) -> int:
    ids = args.ids.split(",") if args.ids else None
    for rid, dest, h, w in decode_to_png(args.archive, args.output, args.size, ids):
        _emit(args, {"record": rid, "file": str(dest), "h": h, "w": w}, f"{rid} -> {dest} ({h}x{w})")
    return 0


def _gather_rasters(inputs):
    files = []
    for item in inputs:
        p = Path(item)
        if p.is_dir():
            files.extend(sorted(q for q in p.iterdir() if q.suffix.lower() in RASTER_SUFFIXES))
        elif p.is_file():
            files.append(p)
        else:
            raise FileNotFoundError(f"no such file or directory: {p}")
    if not files:
        raise RinrError("no raster inputs")
    return files


def _unique_ids(files):
    ids, seen = [], set()
    for i, p in enumerate(files):
        rid = p.stem
        if rid in seen:
            rid = f"{rid}.{i}"
        seen.add(rid)
        ids.append(rid)
    return ids


def _cmd_encode(args) -> int:
    from PIL import Image

    from . import archive, encoder
    from .image import ImageBuffer
    from .net import Architecture
    files = _gather_rasters(args.inputs)
    ids = _unique_ids(files)
    imgs = []
    for p in files:
        with Image.open(p) as im:
            imgs.append(ImageBuffer.from_u8(np.asarray(im.convert("RGB"))))
    try:
        layers, hidden = (int(x) for x in args.arch.split(","))
    except ValueError:
        raise argparse.ArgumentTypeError(f"--arch expects L,H (e.g. 3,15), got {args.arch!r}") from None
    cfg = encoder.EncodeConfig(
        arch=Architecture.uniform(layers, hidden, args.omega), round1_lr=args.round1_lr,
        round1_steps=args.round1_steps, retrain_lr=args.retrain_lr, retrain_steps=args.retrain_steps,
        iterative_prune_ratio=args.iterative_ratio, skip_round2=args.skip_round2, schedule=args.schedule,
        seed=args.seed)
    ds, report = encoder.encode_dataset(imgs, cfg, parallelism=args.jobs, ids=ids, on_error=args.on_error)
    for rec, rep in zip(ds.records, report.per_image):
        _emit(args, {"record": rec.id, "psnr_db": rep.psnr_after_round[-1], "prune_ratio": rep.final_prune_ratio,
                     "seconds": rep.wall_time},
              f"{rec.id}: {rep.psnr_after_round[-1]:.2f} dB, pruned {100 * rep.final_prune_ratio:.1f}%")
    for idx, msg in report.failures:
        print(f"failed: {files[idx]}: {msg}", file=sys.stderr)
    n_bytes = archive.write(ds, args.output)
    _emit(args, {"archive": args.output, "records": len(ds.records), "bytes": n_bytes,
                 "mean_psnr_db": report.mean_psnr, "mean_prune_ratio": report.mean_prune_ratio},
          f"wrote {args.output}: {len(ds.records)} records, {n_bytes} bytes, mean {report.mean_psnr:.2f} dB")
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="rinr-b200", description=__doc__.split("\n\n")[0])
    parser.add_argument("--json", action="store_true", help="JSON-lines output")
    sub = parser.add_subparsers(dest="cmd")
    p = sub.add_parser("decode", help="reconstruct images from an archive (GPU)")
    p.add_argument("archive")
    p.add_argument("-o", "--output", required=True, help="output directory (PNG per record)")
    p.add_argument("--size", type=_parse_size, default=None, help="HxW; defaults to native")
    p.add_argument("--ids", default=None, help="comma-separated record ids")
    p.add_argument("--jobs", type=int, default=1, help="accepted for compatibility; one GPU batch is used")
    p.set_defaults(fn=_cmd_decode)
    p = sub.add_parser("encode", help="fit images and write a .rinr archive (GPU)")
    p.add_argument("inputs", nargs="+", help="image files and/or directories")
    p.add_argument("-o", "--output", required=True)
    p.add_argument("--arch", default="3,15", help="L,H: weight matrices, hidden width")
    p.add_argument("--omega", type=float, default=30.0)
    p.add_argument("--schedule", choices=["cifar", "large"], default="cifar")
    p.add_argument("--skip-round2", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--jobs", type=int, default=1)
    p.add_argument("--round1-lr", type=float, default=5e-4)
    p.add_argument("--round1-steps", type=int, default=5000)
    p.add_argument("--retrain-lr", type=float, default=2e-4)
    p.add_argument("--retrain-steps", type=int, default=10000)
    p.add_argument("--iterative-ratio", type=float, default=0.20)
    p.add_argument("--on-error", choices=["fail_fast", "skip"], default="fail_fast")
    p.set_defaults(fn=_cmd_encode)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        if not getattr(args, "fn", None):
            parser.error("a subcommand is required")
        return args.fn(args)
    except SystemExit as e:
        return int(e.code or 0)
    except BatchItemError as e:
        print(f"rinr-b200: error: {e}", file=sys.stderr)
        return 3 if isinstance(e.cause, NumericError) else 2
    except NumericError as e:
        print(f"rinr-b200: error: {e}", file=sys.stderr)
        return 3
    except (RinrError, OSError, KeyError, argparse.ArgumentTypeError) as e:
        print(f"rinr-b200: error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
