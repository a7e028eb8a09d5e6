"""Model value types of the decode path, mirroring the reference's net.py
(Architecture net.py:24-58, param/weight counts 61-68, LayerWeights 71-79,
InrModel 82-118, validate_model 121-135, init 152-171).

Only the types and the seeded initialiser live here: the forward pass is the
CUDA kernel (``Store.decode`` / ``decoder.decode_batch``).  Objects of the
reference's own classes are accepted anywhere these are (duck-typed).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import TYPE_CHECKING

import numpy as np

from .errors import FormatError, InvalidInputError

if TYPE_CHECKING:
    from .compressor import QuantInfo

DEFAULT_OMEGA = 30.0


@dataclass(frozen=True)
class Architecture:
    """Layer widths including input (2) and output (3), and the sine
    frequency; "N layers" = N weight matrices (net.py:24-34)."""

    dims: tuple
    omega: float = DEFAULT_OMEGA

    def __post_init__(self):
        object.__setattr__(self, "dims", tuple(int(d) for d in self.dims))
        if len(self.dims) < 2:
            raise InvalidInputError("architecture needs at least one weight matrix")
        if self.dims[0] != 2:
            raise InvalidInputError(f"input width must be 2 (x, y), got {self.dims[0]}")
        if self.dims[-1] != 3:
            raise InvalidInputError(f"output width must be 3 (R, G, B), got {self.dims[-1]}")
        if any(d < 1 for d in self.dims):
            raise InvalidInputError(f"every layer width must be >= 1, got {self.dims}")
        if not (self.omega > 0):
            raise InvalidInputError(f"omega must be positive, got {self.omega}")

    @property
    def n_layers(self) -> int:
        return len(self.dims) - 1

    @staticmethod
    def uniform(n_layers: int, hidden: int, omega: float = DEFAULT_OMEGA) -> "Architecture":
        if n_layers < 1:
            raise InvalidInputError("n_layers must be >= 1")
        return Architecture((2, *([hidden] * (n_layers - 1)), 3), omega)


def param_count(arch) -> int:
    """Σ (in·out + out) over weight matrices (net.py:61-63)."""
    d = arch.dims
    return sum(i * o + o for i, o in zip(d[:-1], d[1:]))


def weight_count(arch) -> int:
    """Σ in·out — weight entries only (net.py:66-68)."""
    d = arch.dims
    return sum(i * o for i, o in zip(d[:-1], d[1:]))


@dataclass
class LayerWeights:
    w: np.ndarray  # (out, in)
    b: np.ndarray  # (out,)

    def copy(self) -> "LayerWeights":
        return LayerWeights(self.w.copy(), self.b.copy())


@dataclass
class InrModel:
    """One image's network: weights, pruning masks, optional quantisation
    metadata and the source raster size used as the decode default."""

    arch: Architecture
    layers: list
    mask: list
    source_h: int = 0
    source_w: int = 0
    quant: "QuantInfo | None" = None

    def copy(self) -> "InrModel":
        return InrModel(self.arch, [l.copy() for l in self.layers], [m.copy() for m in self.mask],
                        self.source_h, self.source_w, self.quant)

    @property
    def nnz(self) -> int:
        return int(sum(m.sum() for m in self.mask))

    @property
    def prune_ratio(self) -> float:
        return 1.0 - self.nnz / weight_count(self.arch)


def validate_model(model) -> None:
    """Layer / mask / bias shapes against the architecture (net.py:121-135)."""
    dims = model.arch.dims
    if len(model.layers) != len(dims) - 1 or len(model.mask) != len(dims) - 1:
        raise FormatError(
            f"expected {len(dims) - 1} layers, got {len(model.layers)} layers / {len(model.mask)} masks")
    for i, (lw, m) in enumerate(zip(model.layers, model.mask)):
        want = (dims[i + 1], dims[i])
        if lw.w.shape != want or m.shape != want:
            raise FormatError(f"layer {i}: weight shape {lw.w.shape}, mask {m.shape}, expected {want}")
        if lw.b.shape != (dims[i + 1],):
            raise FormatError(f"layer {i}: bias shape {lw.b.shape}, expected ({dims[i + 1]},)")


def init(arch: Architecture, seed: int, dtype=np.float32) -> InrModel:
    """Seeded sine-network init; identical draws to the reference's net.init
    (net.py:152-171): PCG64(seed), layer 0 U(±1/in), later U(±sqrt(6/in)/ω),
    zero biases, all-ones masks."""
    rng = np.random.default_rng(seed)
    layers, masks = [], []
    for li, (fi, fo) in enumerate(zip(arch.dims[:-1], arch.dims[1:])):
        bound = 1.0 / fi if li == 0 else np.sqrt(6.0 / fi) / arch.omega
        layers.append(LayerWeights(rng.uniform(-bound, bound, size=(fo, fi)).astype(dtype),
                                   np.zeros(fo, dtype=dtype)))
        masks.append(np.ones((fo, fi), dtype=bool))
    return InrModel(arch, layers, masks)
