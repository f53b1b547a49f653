"""KAT (Kolmogorov-Arnold Transformer) built on the B200 group-rational unit.

The caller of the hot path (BASELINE config 4): a ViT whose
MLP is the GR-KAN of the paper -- ``F1 -> W1 -> F2 -> W2`` with the first
group-rational initialised to identity and the second to swish,
8 groups, degrees (5, 4).  Attention, LayerNorm and the linear layers are
stock PyTorch (cuBLAS / SDPA); every rational runs through GroupRationalFn.

``kat_b()`` / ``kat_s()`` / ``kat_t()`` give the paper's three sizes
(patch 16, 224x224 inputs).  ``init_variance_preserving`` follows the
reference code: W ~ N(0, 1 / (alpha * d_in)) with alpha = E[F(z)^2], z ~ N(0, 1)
(pkg/src/grkan/layer.py:282-315).
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F
from torch import nn

from .module import GroupRational, GroupRationalLinearFn, fused_layer_supported


class GRKAN(nn.Module):
    """GR-KAN MLP: rational(identity) -> Linear -> rational(swish) -> Linear.

    ``fused=True`` runs each rational -> Linear pair through
    GroupRationalLinearFn (fused tcgen05 backward) whenever the
    activations qualify (bf16 under autocast, supported shape); otherwise the
    two modules run one after the other.
    """

    def __init__(self, dim: int, hidden: int, groups: int = 8, drop: float = 0.0, fused: bool = False):
        super().__init__()
        self.act1 = GroupRational(groups, init="identity")
        self.fc1 = nn.Linear(dim, hidden)
        self.act2 = GroupRational(groups, init="swish")
        self.fc2 = nn.Linear(hidden, dim)
        self.drop = nn.Dropout(drop)
        self.fused = fused

    def _layer(self, x, act, fc):
        if self.fused and (self.drop.p == 0.0 or not self.training):
            xd = x.to(torch.bfloat16) if x.is_cuda and torch.is_autocast_enabled("cuda") else x
            if fused_layer_supported(xd, act, fc):
                return GroupRationalLinearFn.apply(xd, act.a, act.b, fc.weight, fc.bias)
        return fc(self.drop(act(x)))

    def forward(self, x):
        return self._layer(self._layer(x, self.act1, self.fc1), self.act2, self.fc2)


class Attention(nn.Module):
    def __init__(self, dim: int, heads: int):
        super().__init__()
        self.heads = heads
        self.qkv = nn.Linear(dim, 3 * dim)
        self.proj = nn.Linear(dim, dim)

    def forward(self, x):
        b, n, c = x.shape
        qkv = self.qkv(x).reshape(b, n, 3, self.heads, c // self.heads).permute(2, 0, 3, 1, 4)
        x = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2])
        return self.proj(x.transpose(1, 2).reshape(b, n, c))


class Block(nn.Module):
    def __init__(self, dim: int, heads: int, mlp_ratio: float = 4.0, groups: int = 8, fused: bool = False):
        super().__init__()
        self.norm1 = nn.LayerNorm(dim, eps=1e-6)
        self.attn = Attention(dim, heads)
        self.norm2 = nn.LayerNorm(dim, eps=1e-6)
        self.mlp = GRKAN(dim, int(dim * mlp_ratio), groups, fused=fused)

    def forward(self, x):
        x = x + self.attn(self.norm1(x))
        return x + self.mlp(self.norm2(x))


class KAT(nn.Module):
    def __init__(self, img: int = 224, patch: int = 16, dim: int = 768, depth: int = 12, heads: int = 12,
                 classes: int = 1000, groups: int = 8, fused_mlp: bool = False):
        super().__init__()
        self.patch = nn.Conv2d(3, dim, patch, patch)
        n = (img // patch) ** 2
        self.cls = nn.Parameter(torch.zeros(1, 1, dim))
        self.pos = nn.Parameter(torch.randn(1, n + 1, dim) * 0.02)
        self.blocks = nn.ModuleList([Block(dim, heads, 4.0, groups, fused=fused_mlp) for _ in range(depth)])
        self.norm = nn.LayerNorm(dim, eps=1e-6)
        self.head = nn.Linear(dim, classes)
        init_variance_preserving(self)

    def forward(self, img):
        x = self.patch(img).flatten(2).transpose(1, 2)
        x = torch.cat([self.cls.expand(x.shape[0], -1, -1), x], dim=1) + self.pos
        for blk in self.blocks:
            x = blk(x)
        return self.head(self.norm(x)[:, 0])


def rational_alpha(act: GroupRational, samples: int = 1 << 16, seed: int = 0) -> float:
    """alpha = E[F(z)^2] for z ~ N(0, 1), averaged over groups (layer.py:282-291)."""
    g = torch.Generator().manual_seed(seed)
    z = torch.randn(samples, generator=g, dtype=torch.float64)
    a, b = act.a.detach().double().cpu(), act.b.detach().double().cpu()
    vals = []
    for k in range(a.shape[0]):
        p = torch.zeros_like(z)
        for c in reversed(a[k].tolist()):
            p = p * z + c
        s = torch.zeros_like(z)
        for c in reversed(b[k].tolist()):
            s = s * z + c
        vals.append(float(((p / (1 + (s * z).abs())) ** 2).mean()))
    return sum(vals) / len(vals)


@torch.no_grad()
def init_variance_preserving(model: nn.Module) -> None:
    """GR-KAN linear weights ~ N(0, 1 / (alpha * d_in)), bias 0 (layer.py:293-315)."""
    for m in model.modules():
        if isinstance(m, GRKAN):
            for act, fc in ((m.act1, m.fc1), (m.act2, m.fc2)):
                alpha = rational_alpha(act)
                fc.weight.normal_(0.0, 1.0 / math.sqrt(alpha * fc.in_features))
                fc.bias.zero_()


def kat_t(**kw):
    return KAT(dim=192, depth=12, heads=3, **kw)


def kat_s(**kw):
    return KAT(dim=384, depth=12, heads=6, **kw)


def kat_b(**kw):
    return KAT(dim=768, depth=12, heads=12, **kw)
