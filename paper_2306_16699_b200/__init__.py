"""B200-native batched INR decode (Rapid-INR, arXiv 2306.16699).

Public surface mirrors the reference package ``rinr`` for the decode path
(``decode``, ``decode_batch``, model types, archive writer, errors) and adds
``Store`` — the HBM-resident dataset whose ``decode`` is the fused CUDA
kernel used in a training loop.
"""

from .archive import ArchiveRecord, DatasetArchive, encode_record, serialize, serialize_batch, write
from .compressor import LayerQuant, ModelBatch, QuantInfo, dequantize, prune_l1, quantize
from .errors import (BatchItemError, FormatError, IntegrityError, InvalidInputError, NumericError, RinrError,
                     StructuralError, TrainingError, UnsupportedError)
from .image import ImageBuffer
from .net import Architecture, InrModel, LayerWeights, init, param_count, validate_model, weight_count

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent pieces load lazily so the host-only API (writer, types,
    # archive validation) imports without initialising CUDA.
    if name in ("Store", "pad_crop_params", "resized_crop_params", "IMAGENET_MEAN", "IMAGENET_STD",
                "CIFAR_MEAN", "CIFAR_STD"):
        from . import store
        return getattr(store, name)
    if name in ("bench", "BenchReport"):
        from . import harness
        return getattr(harness, name)
    if name in ("encoder", "transforms", "harness"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    if name in ("decode", "decode_batch", "install"):
        from . import decoder
        return getattr(decoder, name)
    if name in ("read", "ArchiveReader", "materialize", "parse_record", "RawRecord", "RawLayer"):
        from . import reader
        return getattr(reader, name)
    raise AttributeError(name)
