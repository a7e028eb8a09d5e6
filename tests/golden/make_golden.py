"""Generate tests/golden/*.npz by running the REAL reference package.

Run in the build container (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything here calls only the reference's public API (rinr.net.init,
rinr.compressor.prune_l1 / quantize / to_half / dynamic_ratio,
rinr.archive.serialize / read, rinr.decoder.decode_batch, rinr.net.forward,
rinr.net.coordinate_grid).  The fixtures pin:
  * archive bytes written by the reference writer       (our writer, C++ parser)
  * materialised weights per record (archive.read)      (oracle, GPU dequant)
  * decoded pixels at several resolutions (decode_batch) (oracle, GPU decode)
  * forward() on augmented coordinates                   (epilogue checker)
  * coordinate grids                                     (oracle, GPU coords)
"""

from __future__ import annotations

import io
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import rinr  # noqa: E402
from rinr import archive, compressor, decoder, net  # noqa: E402

OUT = Path(__file__).resolve().parent
ARCH_A = net.Architecture((2, 15, 15, 3))
ARCH_C = net.Architecture((2, *([40] * 9), 3))


def r1(m):
    """Last layer w x 20, b = 0.5 (SURVEY §8d 'R1')."""
    m.layers[-1].w = (m.layers[-1].w * np.float32(20.0)).astype(np.float32)
    m.layers[-1].b = np.full_like(m.layers[-1].b, 0.5)
    return m


def cifar_ratios(n, seed):
    rng = np.random.default_rng(seed + 7919)
    sched = compressor.get_schedule("cifar")
    return [compressor.dynamic_ratio(sched, float(p)) for p in rng.uniform(28.0, 37.0, n)]


def ids(n, start=0):
    return [f"img{i:08d}" for i in range(start, start + n)]


def build_archive(models, rid=None):
    rid = rid or ids(len(models))
    recs = [archive.ArchiveRecord(i, m) for i, m in zip(rid, models)]
    buf = io.BytesIO()
    archive.write(archive.DatasetArchive(recs), buf)
    return buf.getvalue()


def flat(model):
    return np.concatenate([np.concatenate([l.w.astype(np.float32).ravel(), l.b.astype(np.float32).ravel()])
                           for l in model.layers])


def store_case(name, data, sizes, n_decode=None):
    arc = archive.read(io.BytesIO(data))
    models = [r.model for r in arc.records]
    P = max(net.param_count(m.arch) for m in models)
    params = np.zeros((len(models), P), np.float32)
    for i, m in enumerate(models):
        f = flat(m)
        params[i, :f.size] = f
    out = {"archive": np.frombuffer(data, np.uint8), "params": params}
    nd = len(models) if n_decode is None else n_decode
    for (h, w) in sizes:
        imgs = decoder.decode_batch(models[:nd], h, w)
        out[f"decode_{h}x{w}"] = np.stack([im.pixels for im in imgs]).astype(np.float32)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: {len(models)} records, {len(data)} bytes, decodes {sizes}")


def main():
    # C1: fp32 dense arch A, literal init (R0) and R1
    store_case("c1_r0", build_archive([_src(net.init(ARCH_A, s)) for s in range(8)]), [(32, 32), (17, 23)])
    store_case("c1_r1", build_archive([_src(r1(net.init(ARCH_A, s))) for s in range(16)]),
               [(32, 32), (1, 1), (1, 7), (9, 1), (64, 48)])
    # C2: R1 + per-record cifar ratio prune + affine8
    ratios = cifar_ratios(32, 0)
    c2 = [compressor.quantize(compressor.prune_l1(_src(r1(net.init(ARCH_A, s))), r), "affine8")
          for s, r in zip(range(32), ratios)]
    store_case("c2", build_archive(c2), [(32, 32), (5, 40)])
    # C3: arch C, R1, 25% prune, affine8 (224x224 in the bench; smaller here)
    c3 = [compressor.quantize(compressor.prune_l1(_src(r1(net.init(ARCH_C, s)), 224, 224), 0.25), "affine8")
          for s in range(3)]
    store_case("c3", build_archive(c3), [(64, 64), (224, 224)], n_decode=2)
    # Encoding zoo: every tag/form/const combination the writer can emit,
    # heterogeneous architectures, odd widths.
    zoo = []
    rng = np.random.default_rng(5)
    for k, dims in enumerate([(2, 15, 15, 3), (2, 1, 3), (2, 8, 3), (2, 5, 7, 3), (2, 32, 32, 32, 3),
                              (2, 40, 40, 3), (2, 16, 16, 3), (2, 33, 3)]):
        m = r1(net.init(net.Architecture(dims, omega=float(rng.choice([30.0, 20.0, 1.5]))), 100 + k))
        for l in m.layers:
            l.b = rng.normal(0, 0.2, l.b.shape).astype(np.float32)
        m = _src(m, int(rng.integers(1, 40)), int(rng.integers(1, 40)))
        kind = k % 4
        if kind == 0:
            m = compressor.quantize(compressor.prune_l1(m, 0.3), "affine16")
        elif kind == 1:
            m = compressor.to_half(compressor.prune_l1(m, 0.05))
        elif kind == 2:
            m = compressor.quantize(compressor.prune_l1(m, 0.1), "affine8")
        else:
            m = compressor.prune_l1(m, 0.45) if len(dims) > 4 else compressor.prune_l1(m, 0.12)
        zoo.append(m)
    # constant hidden layer (degenerate range -> stored as exact f32)
    m = _src(r1(net.init(ARCH_A, 999)))
    m.layers[1].w[:] = np.float32(0.01)
    zoo.append(compressor.quantize(m, "affine8"))
    # sparse + constant: a single kept weight
    m = _src(r1(net.init(ARCH_A, 998)))
    m.mask[1][:] = False
    m.mask[1][3, 4] = True
    m.layers[1].w *= m.mask[1]
    zoo.append(compressor.quantize(m, "affine8"))
    store_case("zoo", build_archive(zoo), [(11, 13), (32, 32)])

    # Epilogue checker: forward() on transformed coordinates (AUG_OFFSET/CROP)
    sys.path.insert(0, str(OUT.parents[1]))
    from oracle import rinr_oracle as O  # noqa: PLC0415
    models = c2[:4]
    aug = {}
    rng = np.random.default_rng(11)
    for i, m in enumerate(models):
        off = [int(rng.integers(0, 9)), int(rng.integers(0, 9)), int(rng.integers(0, 2)), 4, 0]
        crop = [float(np.float32(rng.uniform(0, 0.5))), float(np.float32(rng.uniform(0, 0.5))),
                float(np.float32(rng.uniform(0.3, 0.5))), float(np.float32(rng.uniform(0.3, 0.5))),
                int(rng.integers(0, 2))]
        for mode, params in ((O.AUG_OFFSET, off), (O.AUG_CROP, crop)):
            coords, valid = O.augment_coords(32, 32, mode, params)
            raw = net.forward(m, coords)  # the reference forward at the transformed coordinates
            aug[f"raw_{mode}_{i}"] = raw.astype(np.float32)
            aug[f"valid_{mode}_{i}"] = valid
            aug[f"params_{mode}_{i}"] = np.array(params, np.float32)
    np.savez_compressed(OUT / "augment.npz", **aug)

    grids = {f"grid_{h}x{w}": net.coordinate_grid(h, w) for h, w in
             [(1, 1), (1, 5), (6, 1), (3, 4), (32, 32), (7, 224), (224, 224)]}
    np.savez_compressed(OUT / "grids.npz", **grids)

    # SPEC.md known answers (net.py forward / param_count)
    kat = {
        "param_count": np.array([net.param_count(net.Architecture(d)) for d in
                                 [(2, 1, 3), (2, 15, 15, 3), (2, *([40] * 9), 3)]]),
    }
    m = net.InrModel(net.Architecture((2, 1, 3)), [net.LayerWeights(np.array([[1.0, 0.0]], np.float32),
                                                                     np.zeros(1, np.float32)),
                                                    net.LayerWeights(np.ones((3, 1), np.float32),
                                                                     np.zeros(3, np.float32))],
                     [np.ones((1, 2), bool), np.ones((3, 1), bool)])
    kat["sin15_forward"] = net.forward(m, np.array([[0.5, 0.0]], np.float32))
    np.savez_compressed(OUT / "kat.npz", **kat)
    print("rinr", rinr.__version__, "numpy", np.__version__)


def transforms_case():
    """prune_l1 / quantize / quantize_codes / psnr pinned by the reference
    (checker for csrc/transforms.cu)."""
    from rinr import metrics
    from rinr.image import ImageBuffer
    out = {}
    rng = np.random.default_rng(11)
    cases = []  # (name, model, ratio, scope)
    for s in range(12):
        cases.append((f"a{s}", r1(net.init(ARCH_A, 500 + s)), float(rng.uniform(0.0, 0.6)), "global"))
    # magnitude ties, signed zeros and exact zeros
    m = r1(net.init(ARCH_A, 600))
    for l in m.layers:
        l.w = (np.round(l.w * 64.0) / 64.0).astype(np.float32)
        l.w[0, :2] = np.float32(-0.0)
    cases.append(("ties", m, 0.37, "global"))
    cases.append(("ties_pl", m, 0.37, "per_layer"))
    cases.append(("zero_ratio", r1(net.init(ARCH_A, 601)), 0.0, "global"))
    cases.append(("per_layer", r1(net.init(ARCH_A, 602)), 0.5, "per_layer"))
    cases.append(("structural", r1(net.init(ARCH_A, 603)), 0.999, "global"))
    cases.append(("archc", r1(net.init(ARCH_C, 604)), 0.25, "global"))
    names = []
    for name, m, ratio, scope in cases:
        names.append(name)
        out[f"{name}/dims"] = np.array(m.arch.dims, np.int32)
        out[f"{name}/ratio"] = np.float64(ratio)
        out[f"{name}/scope"] = np.array(scope)
        out[f"{name}/w"] = np.concatenate([l.w.ravel() for l in m.layers]).view(np.uint32)
        out[f"{name}/b"] = np.concatenate([l.b.ravel() for l in m.layers])
        out[f"{name}/mask"] = np.concatenate([x.ravel() for x in m.mask]).astype(np.uint8)
        try:
            p = compressor.prune_l1(m, ratio, scope=scope)
        except Exception as e:  # noqa: BLE001
            out[f"{name}/prune_error"] = np.array(type(e).__name__)
            continue
        out[f"{name}/pw"] = np.concatenate([l.w.ravel() for l in p.layers]).view(np.uint32)
        out[f"{name}/pmask"] = np.concatenate([x.ravel() for x in p.mask]).astype(np.uint8)
        for mode in ("affine8", "affine16"):
            q = compressor.quantize(p, mode)
            out[f"{name}/{mode}/w"] = np.concatenate([l.w.ravel() for l in q.layers]).view(np.uint32)
            lay = sorted(q.quant.layers)
            out[f"{name}/{mode}/scale"] = np.array([q.quant.layers[i].scale for i in lay], np.float64)
            out[f"{name}/{mode}/zp"] = np.array([q.quant.layers[i].zero_point for i in lay], np.int64)
            out[f"{name}/{mode}/const"] = np.array([q.quant.layers[i].constant for i in lay], bool)
            for i in lay:
                if not q.quant.layers[i].constant:
                    out[f"{name}/{mode}/codes{i}"] = compressor.quantize_codes(q, i).ravel().astype(np.uint16)
    # quantize edge cases on hand-built masks: an all-masked hidden layer
    # (kept.size == 0) and a constant kept range
    m = r1(net.init(ARCH_A, 605))
    m.mask[1][:] = False
    m.layers[1].w[:] = 0.0
    m.mask[1][3, 4] = True
    m.layers[1].w[3, 4] = np.float32(0.25)
    names.append("qedge")
    out["qedge/dims"] = np.array(m.arch.dims, np.int32)
    out["qedge/w"] = np.concatenate([l.w.ravel() for l in m.layers]).view(np.uint32)
    out["qedge/b"] = np.concatenate([l.b.ravel() for l in m.layers])
    out["qedge/mask"] = np.concatenate([x.ravel() for x in m.mask]).astype(np.uint8)
    q = compressor.quantize(m, "affine8")
    out["qedge/affine8/w"] = np.concatenate([l.w.ravel() for l in q.layers]).view(np.uint32)
    out["qedge/affine8/const"] = np.array([q.quant.layers[1].constant], bool)
    out["names"] = np.array(names)
    # PSNR: decoded images vs perturbed targets, float and u8 paths
    ims = decoder.decode_batch([_src(r1(net.init(ARCH_A, 700 + s))) for s in range(4)])
    a = np.stack([im.pixels for im in ims])
    b = np.clip(a + rng.normal(0, 0.02, a.shape).astype(np.float32), 0, 1).astype(np.float32)
    b[3] = a[3]
    out["psnr/a"], out["psnr/b"] = a, b
    out["psnr/f"] = np.array([metrics.psnr(ImageBuffer(x), ImageBuffer(y)).psnr_db for x, y in zip(a, b)])
    out["psnr/q"] = np.array([metrics.psnr(ImageBuffer(x), ImageBuffer(y), quantized=True).psnr_db
                              for x, y in zip(a, b)])
    np.savez_compressed(OUT / "transforms.npz", **out)


def test_images(n, h, w, seed):
    """Smooth deterministic RGB test images in [0, 1] (f32)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.linspace(0, 1, h), np.linspace(0, 1, w), indexing="ij")
    out = []
    for _ in range(n):
        img = np.zeros((h, w, 3), np.float64)
        for c in range(3):
            for _ in range(3):
                fx, fy, ph = rng.uniform(0.5, 4.0), rng.uniform(0.5, 4.0), rng.uniform(0, 2 * np.pi)
                img[..., c] += rng.uniform(0.1, 0.3) * np.sin(2 * np.pi * (fx * xx + fy * yy) + ph)
        out.append(np.clip(0.5 + img, 0.0, 1.0).astype(np.float32))
    return np.stack(out)


def encoder_case():
    """net.loss_and_grad / Adam / encoder._train / fit_round1 / fit_full pinned
    by the reference (checker for the GPU encoder)."""
    from rinr import encoder
    from rinr.image import ImageBuffer
    out = {}
    imgs = test_images(3, 16, 16, seed=21)
    out["images16"] = imgs
    coords = net.coordinate_grid(16, 16)
    # (1) loss + gradients: fresh init, and a pruned + perturbed model
    for k, seed in enumerate((31, 32)):
        m = net.init(ARCH_A, seed)
        if k == 1:
            m = compressor.prune_l1(m, 0.3)
            for l in m.layers:
                l.b[:] = np.random.default_rng(seed).normal(0, 0.05, l.b.shape).astype(np.float32)
        loss, grads = net.loss_and_grad(m, coords, imgs[k].reshape(-1, 3))
        out[f"grad{k}/seed"] = np.int64(seed)
        out[f"grad{k}/w"] = np.concatenate([l.w.ravel() for l in m.layers])
        out[f"grad{k}/b"] = np.concatenate([l.b.ravel() for l in m.layers])
        out[f"grad{k}/mask"] = np.concatenate([x.ravel() for x in m.mask]).astype(np.uint8)
        out[f"grad{k}/loss"] = np.float64(loss)
        out[f"grad{k}/gw"] = np.concatenate([g.w.ravel() for g in grads])
        out[f"grad{k}/gb"] = np.concatenate([g.b.ravel() for g in grads])
    # (2) _train: 40 steps from init on image 2
    m = net.init(ARCH_A, 33)
    curve = []
    encoder._train(m, coords, imgs[2].reshape(-1, 3), 5e-4, 40, curve)
    out["train/curve"] = np.array(curve)
    out["train/w"] = np.concatenate([l.w.ravel() for l in m.layers])
    out["train/b"] = np.concatenate([l.b.ravel() for l in m.layers])
    # (3) fit_round1 / fit_full on 32x32 images with shortened schedules
    imgs32 = test_images(2, 32, 32, seed=22)
    out["images32"] = imgs32
    cfg1 = encoder.EncodeConfig(ARCH_A, round1_steps=300, seed=encoder.derive_seed(7, 0))
    m1, r1_ = encoder.fit_round1(ImageBuffer(imgs32[0]), cfg1)
    out["round1/seed"] = np.int64(cfg1.seed)
    out["round1/psnr"] = np.array(r1_.psnr_after_round)
    out["round1/curve"] = np.array(r1_.loss_curve)
    cfgf = encoder.EncodeConfig(ARCH_A, round1_steps=200, retrain_steps=100, seed=encoder.derive_seed(7, 1))
    mf, rf = encoder.fit_full(ImageBuffer(imgs32[1]), cfgf)
    out["full/seed"] = np.int64(cfgf.seed)
    out["full/psnr"] = np.array(rf.psnr_after_round)
    out["full/psnr_mask"] = np.array(rf.psnr_after_mask)
    out["full/ratio"] = np.float64(rf.final_prune_ratio)
    out["derive_seed"] = np.array([encoder.derive_seed(s, i) for s in (0, 7, 2**40) for i in (0, 1, 999)],
                                  np.uint64)
    # (4) wide / deep nets (the general GPU encoder): loss_and_grad of the
    # Mini-ImageNet arch [2,40x9,3] (fresh and pruned) and 20 _train steps of
    # a 4-layer 32-wide net, on 12x12 images
    imgs12 = test_images(2, 12, 12, seed=23)
    out["images12"] = imgs12
    c12 = net.coordinate_grid(12, 12)
    for k, seed in enumerate((41, 42)):
        m = net.init(ARCH_C, seed)
        if k == 1:
            m = compressor.prune_l1(m, 0.3)
            for l in m.layers:
                l.b[:] = np.random.default_rng(seed).normal(0, 0.02, l.b.shape).astype(np.float32)
        loss, grads = net.loss_and_grad(m, c12, imgs12[k].reshape(-1, 3))
        out[f"wgrad{k}/w"] = np.concatenate([l.w.ravel() for l in m.layers])
        out[f"wgrad{k}/b"] = np.concatenate([l.b.ravel() for l in m.layers])
        out[f"wgrad{k}/mask"] = np.concatenate([x.ravel() for x in m.mask]).astype(np.uint8)
        out[f"wgrad{k}/loss"] = np.float64(loss)
        out[f"wgrad{k}/gw"] = np.concatenate([g.w.ravel() for g in grads])
        out[f"wgrad{k}/gb"] = np.concatenate([g.b.ravel() for g in grads])
    arch_d = net.Architecture((2, 32, 32, 32, 3))
    m = net.init(arch_d, 44)
    curve = []
    encoder._train(m, c12, imgs12[1].reshape(-1, 3), 2e-4, 20, curve)
    out["wtrain/curve"] = np.array(curve)
    out["wtrain/w"] = np.concatenate([l.w.ravel() for l in m.layers])
    np.savez_compressed(OUT / "encoder.npz", **out)


def fitted_case():
    """INRs actually fitted by the reference encoder (encoder.fit_round1),
    then compressed the paper's way (prune_l1 to the dynamic ratio or 25%,
    quantize affine8), written by the reference writer.
    Pins the PSNR against the SOURCE image of the reference decode of every
    stored record, so the GPU decode's bf16 / fp32 paths can be held to
    |PSNR(gpu, source) - PSNR(ref, source)| <= 0.05 dB."""
    from rinr import encoder, metrics
    from rinr.image import ImageBuffer
    out = {}
    sched = compressor.get_schedule("cifar")
    for name, arch, n, size, steps in (("A", ARCH_A, 4, 32, 3000), ("C", ARCH_C, 2, 48, 600)):
        imgs = test_images(n, size, size, seed=41 if name == "A" else 42)
        models = []
        for i in range(n):
            cfg = encoder.EncodeConfig(arch, round1_steps=steps, seed=encoder.derive_seed(9, i))
            m, rep = encoder.fit_round1(ImageBuffer(imgs[i]), cfg)
            models.append(m)  # dense f32 as fitted
            ratio = compressor.dynamic_ratio(sched, rep.psnr_after_round[0]) if name == "A" else 0.25
            models.append(compressor.quantize(compressor.prune_l1(m, ratio), "affine8"))
        data = build_archive(models)
        recs = archive.read(io.BytesIO(data)).records
        dec = decoder.decode_batch([r.model for r in recs])
        src = np.repeat(imgs, 2, axis=0)  # record 2i, 2i+1 encode image i
        out[f"{name}/archive"] = np.frombuffer(data, np.uint8)
        out[f"{name}/source"] = src
        out[f"{name}/decode"] = np.stack([d.pixels for d in dec])
        out[f"{name}/psnr"] = np.array([metrics.psnr(d, ImageBuffer(s)).psnr_db for d, s in zip(dec, src)])
    np.savez_compressed(OUT / "fitted.npz", **out)


def digest_case():
    """rinr.bench.bench digests (sha256 over the decoded u8 pixels, record
    order, bench.py:41-73) of the golden stores, plus one sha256 per record,
    so the GPU harness's digest can be pinned to the reference's."""
    import hashlib
    import tempfile
    from rinr import bench as rbench
    out = {}
    for case in ("c1_r0", "c1_r1", "c2", "zoo", "fitted_A"):
        if case == "fitted_A":
            data = np.load(OUT / "fitted.npz")["A/archive"].tobytes()
        else:
            data = np.load(OUT / f"{case}.npz")["archive"].tobytes()
        with tempfile.NamedTemporaryFile(suffix=".rinr") as f:
            f.write(data)
            f.flush()
            rep = rbench.bench(f.name, batch=4)
        out[f"{case}/digest"] = np.array(rep.digest)
        recs = archive.read(io.BytesIO(data)).records
        per = [hashlib.sha256(decoder.decode(r.model).as_u8().tobytes()).hexdigest() for r in recs]
        out[f"{case}/per_record"] = np.array(per)
    np.savez_compressed(OUT / "digests.npz", **out)


def _src(m, h=32, w=32):
    m.source_h, m.source_w = h, w
    return m


if __name__ == "__main__" and sys.argv[1:] == ["transforms"]:
    transforms_case()
elif __name__ == "__main__" and sys.argv[1:] == ["encoder"]:
    encoder_case()
elif __name__ == "__main__" and sys.argv[1:] == ["fitted"]:
    fitted_case()
elif __name__ == "__main__" and sys.argv[1:] == ["digests"]:
    digest_case()
elif __name__ == "__main__":
    main()
    transforms_case()
    encoder_case()
    fitted_case()
    digest_case()
