"""Shared helpers for the transform parity tests (golden: tests/golden/transforms.npz)."""

import numpy as np


def split(flat, dims, dtype=None):
    """Flat concatenated matrices -> list of (out, in) arrays."""
    out, off = [], 0
    for l in range(len(dims) - 1):
        sz = int(dims[l] * dims[l + 1])
        x = flat[off:off + sz].reshape(int(dims[l + 1]), int(dims[l]))
        out.append(x.astype(dtype) if dtype is not None else x)
        off += sz
    return out


def split_bias(flat, dims):
    out, off = [], 0
    for l in range(len(dims) - 1):
        out.append(flat[off:off + int(dims[l + 1])])
        off += int(dims[l + 1])
    return out


def case(g, name):
    dims = g[f"{name}/dims"]
    w = split(g[f"{name}/w"].view(np.float32), dims)
    m = split(g[f"{name}/mask"], dims, bool)
    b = split_bias(g[f"{name}/b"], dims)
    return dims, w, m, b


def cat(mats):
    return np.concatenate([x.ravel() for x in mats])


def smooth_images(n, h, w, seed):
    """Smooth deterministic RGB images in [0, 1] (f32) — the generator
    tests/golden/make_golden.py uses for the encoder fixtures."""
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
