"""The decode's consumer (BASELINE configs 4 and 5): a
ResNet-18 training loop whose every batch is decoded on the fly from an
HBM-resident INR store (the whole dataset stays in device
memory as INRs; ResNet-18, SGD lr 1e-2, weight decay 5e-4).

Multi-GPU follows the path's natural partition: the store is sharded by
record (``Store(..., shard_rank, shard_world)`` keeps records k % world ==
rank), each rank samples its batches from a per-epoch permutation of its own
shard, decodes them locally, and the only collective is DDP's gradient
all-reduce (NCCL over NVLink; gloo in the CPU-side tests).  Labels are
synthetic and fixed per record (global index mod classes).
"""

from __future__ import annotations

import numpy as np
import torch

from . import synth
from .store import (CIFAR_MEAN, CIFAR_STD, IMAGENET_MEAN, IMAGENET_STD, Store, pad_crop_params,
                    resized_crop_params)
from .trace import stage


def open_sharded_store(config: str, total: int, rank: int, world: int, device="cuda", seed: int = 4242) -> Store:
    """Every rank builds the same `total`-record archive (GPU generator, so
    identical bytes on every rank) and keeps its shard."""
    data = synth.gpu_store_bytes(config, total, seed=seed, device=device)
    return Store(data, device=device, shard_rank=rank, shard_world=world)


class DecodeTrainLoop:
    """One training step = sample ids from the local shard, decode them with
    crop/flip/normalise into a bf16 NCHW batch (one fused launch), then a
    ResNet-18 forward/backward/SGD step (optionally DDP-wrapped)."""

    def __init__(self, store: Store, h: int, w: int, batch: int, classes: int = 10, precision: str = "bf16",
                 aug: str = "crop", seed: int = 0, ddp: bool = False, device="cuda", lr: float = 1e-2,
                 weight_decay: float = 5e-4, model: torch.nn.Module | None = None):
        import torchvision  # noqa: PLC0415
        self.st = store
        self.dev = torch.device(device)
        self.h, self.w, self.batch, self.classes = h, w, batch, classes
        self.aug = aug
        mean, std = (IMAGENET_MEAN, IMAGENET_STD) if aug == "crop" else (CIFAR_MEAN, CIFAR_STD)
        self.params = store.decode_params(h, w, dtype=torch.bfloat16, precision=precision, aug_mode=aug, mean=mean,
                                          std=std)
        net = model if model is not None else torchvision.models.resnet18(num_classes=classes)
        net = net.to(self.dev).to(memory_format=torch.channels_last)
        if ddp:
            net = torch.nn.parallel.DistributedDataParallel(
                net, device_ids=[self.dev.index] if self.dev.type == "cuda" else None)
        self.model = net
        self.opt = torch.optim.SGD(net.parameters(), lr=lr, momentum=0.9, weight_decay=weight_decay)
        self.lossf = torch.nn.CrossEntropyLoss()
        # sampling and augmentation parameters are drawn on the device: a step
        # issues no host->device copies and never waits on the host
        self.gen = torch.Generator(device=self.dev).manual_seed(seed)
        n = len(store)
        rank, world = int(store.info.shard_rank), int(store.info.shard_world)
        glob = torch.arange(n, dtype=torch.int64) * world + rank  # global record index of local i
        self.labels_all = (glob % classes).to(self.dev)
        self.perm = torch.empty(0, dtype=torch.int64, device=self.dev)
        self.pos = 0
        self.x = torch.empty((batch, 3, h, w), dtype=torch.bfloat16, device=self.dev)

    def next_ids(self) -> torch.Tensor:
        """The next batch of local ids: a fresh permutation of the shard per epoch."""
        n = len(self.st)
        if self.pos + self.batch > self.perm.numel():
            self.perm = torch.randperm(n, generator=self.gen, device=self.dev)
            self.pos = 0
        ids = self.perm[self.pos:self.pos + self.batch]
        self.pos += self.batch
        return ids

    def next_aug(self) -> torch.Tensor:
        if self.aug == "crop":
            return resized_crop_params(self.batch, generator=self.gen)
        return pad_crop_params(self.batch, 4, generator=self.gen)

    def decode(self, ids: torch.Tensor, aug: torch.Tensor) -> torch.Tensor:
        self.st.decode(ids, out=self.x, aug=aug, params=self.params, check=False)
        return self.labels_all[ids]

    def train_on(self, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        with stage("train.forward"), torch.autocast(self.dev.type, dtype=torch.bfloat16,
                                                     enabled=self.dev.type == "cuda"):
            loss = self.lossf(self.model(x.contiguous(memory_format=torch.channels_last)), y)
        self.opt.zero_grad(set_to_none=True)
        with stage("train.backward"):  # includes DDP's bucketed gradient all-reduce
            loss.backward()
        with stage("train.sgd"):
            self.opt.step()
        return loss.detach()

    def step(self) -> torch.Tensor:
        y = self.decode(self.next_ids(), self.next_aug())
        return self.train_on(self.x, y)

    def _timed(self, fn, k: int) -> float:
        torch.cuda.synchronize(self.dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize(self.dev)
        return e0.elapsed_time(e1) * 1e-3

    def time_decode_only(self, k: int) -> float:
        batches = [(self.next_ids(), self.next_aug()) for _ in range(k)]
        it = iter(batches)
        return self._timed(lambda: self.decode(*next(it)), k)

    def time_train_only(self, k: int) -> float:
        y = self.decode(self.next_ids(), self.next_aug())
        return self._timed(lambda: self.train_on(self.x, y), k)


def param_checksum(model: torch.nn.Module) -> np.ndarray:
    """f64 sum and sum of squares of every parameter (replica-identity checks)."""
    m = model.module if hasattr(model, "module") else model
    with torch.no_grad():
        flat = torch.cat([p.detach().double().reshape(-1) for p in m.parameters()])
    return np.array([float(flat.sum()), float((flat * flat).sum())])
