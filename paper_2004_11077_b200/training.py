"""Config 5 of BASELINE.json: ResNet-18 (32x32-input variant) whose 3x3 stride-1 convolutions are
the quantized Winograd-aware layer, one training step (forward, STE backward, SGD momentum 0.9),
data parallel over N GPUs with one NCCL gradient all-reduce per step.

Also the batch-sharding helpers used by bench.py for the inference configs (each rank an
independent call on its own shard, no collective).
"""

from __future__ import annotations

import os
from typing import Callable

import torch
import torch.nn as nn
import torch.nn.functional as F

from .layer import WinogradAwareConv2d
from .quantize import QuantConfig


def winograd_conv_factory(mode: str = "legendre", qconfig: QuantConfig | None = None,
                          scale_groups: str = "image") -> Callable[[int, int], nn.Module]:
    q = QuantConfig.uniform(8) if qconfig is None else qconfig

    def make(cin: int, cout: int) -> nn.Module:
        return WinogradAwareConv2d(cin, cout, padding=1, bias=False, mode=mode, qconfig=q, scale_groups=scale_groups)

    return make


def plain_conv_factory(cin: int, cout: int) -> nn.Module:
    """fp32 3x3 convolution with the same interface (used only by CPU tests of the DDP plumbing)."""
    return nn.Conv2d(cin, cout, 3, padding=1, bias=False)


class BasicBlock(nn.Module):
    def __init__(self, cin: int, cout: int, stride: int, conv3: Callable[[int, int], nn.Module]):
        super().__init__()
        # stride-1 3x3 convolutions run on the Winograd layer; stride-2 and 1x1 stay in PyTorch
        self.conv1 = conv3(cin, cout) if stride == 1 else nn.Conv2d(cin, cout, 3, stride, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(cout)
        self.conv2 = conv3(cout, cout)
        self.bn2 = nn.BatchNorm2d(cout)
        self.shortcut = nn.Sequential()
        if stride != 1 or cin != cout:
            self.shortcut = nn.Sequential(nn.Conv2d(cin, cout, 1, stride, bias=False), nn.BatchNorm2d(cout))

    def forward(self, x):
        out = F.relu(self.bn1(self.conv1(x)))
        out = self.bn2(self.conv2(out))
        return F.relu(out + self.shortcut(x))


class ResNet18(nn.Module):
    """CIFAR-style ResNet-18: 3x3 stem, stages 64/128/256/512, global pool, 10-way FC."""

    def __init__(self, conv3: Callable[[int, int], nn.Module], num_classes: int = 10):
        super().__init__()
        self.stem = conv3(3, 64)
        self.bn = nn.BatchNorm2d(64)
        cfg = [(64, 1), (128, 2), (256, 2), (512, 2)]
        layers, cin = [], 64
        for cout, stride in cfg:
            layers += [BasicBlock(cin, cout, stride, conv3), BasicBlock(cout, cout, 1, conv3)]
            cin = cout
        self.layers = nn.Sequential(*layers)
        self.fc = nn.Linear(512, num_classes)

    def forward(self, x):
        x = F.relu(self.bn(self.stem(x)))
        x = self.layers(x)
        x = F.adaptive_avg_pool2d(x, 1).flatten(1)
        return self.fc(x)


def count_winograd_layers(model: nn.Module) -> int:
    return sum(1 for m in model.modules() if isinstance(m, WinogradAwareConv2d))


def synthetic_batch(batch: int, rank: int, seed: int = 0, device="cpu"):
    """Config-5 data: images ~ N(0,1) [batch,3,32,32], labels uniform in [0,10); rank-seeded."""
    g = torch.Generator(device="cpu")
    g.manual_seed(seed * 1000003 + rank)
    x = torch.randn(batch, 3, 32, 32, generator=g)
    y = torch.randint(0, 10, (batch,), generator=g)
    return x.to(device), y.to(device)


def make_optimizer(model: nn.Module, lr: float = 0.1) -> torch.optim.Optimizer:
    return torch.optim.SGD(model.parameters(), lr=lr, momentum=0.9)


def train_step(model: nn.Module, opt: torch.optim.Optimizer, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """One step: forward, STE backward (gradients all-reduced by DDP), SGD momentum update."""
    opt.zero_grad(set_to_none=True)
    loss = F.cross_entropy(model(x), y)
    loss.backward()
    opt.step()
    return loss.detach()


def invalidate_weight_caches(model: nn.Module) -> None:
    """Forget every cached weight transform (after graph replays updated the weights without Python seeing it)."""
    for m in model.modules():
        if isinstance(m, WinogradAwareConv2d):
            for r in m._runners.values():
                r.wcache.key = None


def make_graphed_step(model: nn.Module, opt: torch.optim.Optimizer, x: torch.Tensor, y: torch.Tensor,
                      warmup: int = 3):
    """The whole training step (forward, STE backward, SGD update) captured once as a CUDA graph: the ~50
    kernel launches and ctypes calls of each of the 14 Winograd layers are launch-bound at batch 256, and
    a replay issues them without any host work.  Single-process only (no DDP hooks inside the capture).
    Returns `step()` -> loss tensor (static: overwritten by every replay).  x and y are the static inputs:
    copy new batches into them.  Call invalidate_weight_caches(model) before going back to eager calls."""
    side = torch.cuda.Stream(device=x.device)
    side.wait_stream(torch.cuda.current_stream(x.device))
    with torch.cuda.stream(side):  # eager warm-up: allocations, momentum buffers, per-device kernel attributes
        for _ in range(warmup):
            train_step(model, opt, x, y)
    torch.cuda.current_stream(x.device).wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    opt.zero_grad(set_to_none=True)
    with torch.cuda.graph(graph):
        loss = F.cross_entropy(model(x), y)
        loss.backward()
        opt.step()
    loss_out = loss.detach()

    def step() -> torch.Tensor:
        graph.replay()
        return loss_out

    return step


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [start, stop) of `total` items for `rank` (sizes differ by at most one)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def dist_env() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))
