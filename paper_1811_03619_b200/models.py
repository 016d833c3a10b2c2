"""Models whose gradients feed the hot path, bound to flat fp32 buffers.

The engine exchanges ONE flat gradient vector per iteration, exactly like the
reference (`ModelSpec.param_blocks`, /root/reference/pkg/src/gradpipe/models.py:57-66,
"parameters and gradients live in flat float32 vectors"). `FlatModel` binds a
torch module's parameters and gradients as views into two contiguous CUDA
buffers, so the backward pass writes the gradient straight into the buffer
the ring kernel reads — no flatten/unflatten copies on the critical path.

Model families (BASELINE.json configs):
  * logistic / MLP with the reference's exact flat layout (W stored
    (d_in, d_out) row-major, then b; models.py:57-66) and init (:84-102) — C1
  * SmallCNN — CIFAR-10-shaped 3-conv + 2-FC network (the paper's
    "AlexNet-style CIFAR" net) — C2
  * AlexNet (61,100,840 params) and ResNet-50 (25,557,032) from torchvision,
    randomly initialised — C3 / C4
Forward/backward run in torch/cuDNN (not the product: SURVEY §2 marks the
models as gradient sources, the hot path starts at the flat gradient).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from .errors import ConfigError

LOGISTIC, MLP = "logistic", "mlp"


@dataclass(frozen=True)
class ModelSpec:
    """Same fields and layout as gradpipe.models.ModelSpec (models.py:29-73)."""

    kind: str
    layer_dims: tuple

    def __post_init__(self):
        if self.kind not in (LOGISTIC, MLP):
            raise ConfigError(f"unknown model kind {self.kind!r}")
        if len(self.layer_dims) < 2 or any(d < 1 for d in self.layer_dims):
            raise ConfigError(f"bad layer dims {self.layer_dims}")
        if self.kind == LOGISTIC and len(self.layer_dims) != 2:
            raise ConfigError("logistic model takes exactly (input_dim, num_classes)")

    @property
    def num_classes(self) -> int:
        return self.layer_dims[-1]

    @property
    def input_dim(self) -> int:
        return self.layer_dims[0]

    def param_blocks(self):
        blocks, off = [], 0
        for d_in, d_out in zip(self.layer_dims[:-1], self.layer_dims[1:]):
            blocks.append((off, (d_in, d_out)))
            off += d_in * d_out
            blocks.append((off, (d_out,)))
            off += d_out
        return blocks

    @property
    def num_params(self) -> int:
        return sum((a + 1) * b for a, b in zip(self.layer_dims[:-1], self.layer_dims[1:]))


def logistic_model(input_dim: int, num_classes: int) -> ModelSpec:
    return ModelSpec(LOGISTIC, (input_dim, num_classes))


def mlp_model(input_dim: int, hidden, num_classes: int) -> ModelSpec:
    return ModelSpec(MLP, (input_dim, *hidden, num_classes))


def init_params(spec: ModelSpec, seed: int = 0) -> np.ndarray:
    """models.py:84-102: zeros; MLP weights uniform(+-sqrt(6/(fan_in+fan_out)))
    drawn from default_rng(seed) block by block, biases zero."""
    w = np.zeros(spec.num_params, np.float32)
    if spec.kind == MLP:
        g = np.random.default_rng(seed)
        for off, shape in spec.param_blocks():
            if len(shape) == 2:
                lim = np.sqrt(6.0 / (shape[0] + shape[1]))
                w[off:off + shape[0] * shape[1]] = g.uniform(-lim, lim, size=shape).reshape(-1).astype(np.float32)
    return w


class SpecNet(nn.Module):
    """Logistic regression / ReLU MLP with the reference's parameter layout:
    z = a @ W + b with W of shape (d_in, d_out) (models.py:118-131)."""

    def __init__(self, spec: ModelSpec):
        super().__init__()
        self.spec = spec
        ps = []
        for _, shape in spec.param_blocks():
            ps.append(nn.Parameter(torch.zeros(shape)))
        self.ps = nn.ParameterList(ps)

    def forward(self, x):
        n = len(self.ps) // 2
        for i in range(n):
            x = x @ self.ps[2 * i] + self.ps[2 * i + 1]
            if i < n - 1:
                x = F.relu(x)
        return x


class SmallCNN(nn.Module):
    """CIFAR-10-shaped 3 conv + 2 FC net ("3 convolutional
    layers and 2 fully connected layers followed by a softmax")."""

    def __init__(self, num_classes: int = 10):
        super().__init__()
        self.c1 = nn.Conv2d(3, 64, 5, padding=2)
        self.c2 = nn.Conv2d(64, 128, 5, padding=2)
        self.c3 = nn.Conv2d(128, 256, 3, padding=1)
        self.f1 = nn.Linear(256 * 4 * 4, 1024)
        self.f2 = nn.Linear(1024, num_classes)

    def forward(self, x):
        x = F.max_pool2d(F.relu(self.c1(x)), 2)
        x = F.max_pool2d(F.relu(self.c2(x)), 2)
        x = F.max_pool2d(F.relu(self.c3(x)), 2)
        x = F.relu(self.f1(x.flatten(1)))
        return self.f2(x)


def build_torch_model(name: str) -> tuple[nn.Module, tuple, int]:
    """(module, per-sample input shape, classes) for a BASELINE config name."""
    name = name.lower()
    if name in ("mlp", "mnist_mlp", "c1"):
        return SpecNet(mlp_model(784, (500, 500), 10)), (784,), 10
    if name in ("small_cnn", "cifar_cnn", "c2"):
        return SmallCNN(10), (3, 32, 32), 10
    if name in ("alexnet", "c3"):
        import torchvision
        return torchvision.models.alexnet(num_classes=1000), (3, 224, 224), 1000
    if name in ("resnet50", "c4"):
        import torchvision
        return torchvision.models.resnet50(num_classes=1000), (3, 224, 224), 1000
    raise ConfigError(f"unknown model {name!r}")


def full_fp32_math() -> None:
    """Disable TF32 for cuDNN convolutions and cuBLAS matmuls.

    torch enables TF32 convolutions by default (cudnn.allow_tf32=True), a
    10-bit-mantissa product; the reference computes its models in float32 /
    float64 (models.py:118-195), so the engine runs every model in full fp32."""
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.set_float32_matmul_precision("highest")


class FlatModel:
    """A module whose parameters/gradients are views into flat CUDA buffers.

    `params` and `grads` are 1-D fp32 tensors of num_params elements, 256-byte
    aligned; parameter order is module.parameters() order (for SpecNet that
    is exactly the reference's flat layout)."""

    def __init__(self, module: nn.Module, device, init_flat: np.ndarray | None = None, grad_buffers: int = 1):
        full_fp32_math()
        self.module = module.to(device)
        self.plist = [p for p in self.module.parameters() if p.requires_grad]
        self.num_params = sum(p.numel() for p in self.plist)
        self.params = torch.empty(self.num_params, dtype=torch.float32, device=device)
        # K flat gradient buffers: the fused ring reads buffer t % K while the
        # next backward writes another one
        self.grad_bufs = [torch.zeros(self.num_params, dtype=torch.float32, device=device)
                          for _ in range(max(1, grad_buffers))]
        self._grad_views = [[] for _ in self.grad_bufs]
        off = 0
        for p in self.plist:
            k = p.numel()
            view = self.params[off:off + k].view_as(p)
            view.copy_(p.data)
            p.data = view
            for i, g in enumerate(self.grad_bufs):
                self._grad_views[i].append(g[off:off + k].view_as(p))
            off += k
        self.use_grad_buffer(0)
        if init_flat is not None:
            if init_flat.size != self.num_params:
                raise ConfigError(f"init vector has {init_flat.size} values, model has {self.num_params}")
            self.params.copy_(torch.from_numpy(np.ascontiguousarray(init_flat, np.float32)))

    def ensure_grad_buffers(self, k: int) -> None:
        while len(self.grad_bufs) < k:
            g = torch.zeros(self.num_params, dtype=torch.float32, device=self.params.device)
            views, off = [], 0
            for p in self.plist:
                views.append(g[off:off + p.numel()].view_as(p))
                off += p.numel()
            self.grad_bufs.append(g)
            self._grad_views.append(views)

    def use_grad_buffer(self, i: int) -> torch.Tensor:
        """Point every parameter's .grad at flat buffer i (autograd accumulates
        in place into an existing .grad, so backward writes straight into it)."""
        self._cur = i
        for p, v in zip(self.plist, self._grad_views[i]):
            p.grad = v
        return self.grad_bufs[i]

    @property
    def grads(self) -> torch.Tensor:
        return self.grad_bufs[self._cur]

    def zero_grad(self):
        self.grads.zero_()

    def loss_and_grad(self, x, y, zero: bool = True):
        """Mean softmax cross-entropy; gradient lands in self.grads (autograd
        accumulates into it: zero=False when the caller guarantees the buffer
        is already zero -- the engine clears it on the comm stream right after
        the ring has read it, off the compute stream's critical path)."""
        if zero:
            self.grads.zero_()
        logits = self.module(x)
        loss = F.cross_entropy(logits, y)
        loss.backward()
        return loss.detach()
