"""Random-init bf16 weights of the target and the drafter (there are no checkpoints).

Layout is the kernels' layout: nn.Linear [out, in] row-major, q|k|v and
gate|up fused along the output dimension.  Init N(0, std^2) from a seeded CUDA
generator; norm weights are 1 (drafter final norm = logit_scale).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .config import DrafterConfig, ModelConfig

STD = 0.02


def _normal(shape, g, dev) -> torch.Tensor:
    t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
    t.normal_(0.0, STD, generator=g)
    return t


def _ones(n, dev, value: float = 1.0) -> torch.Tensor:
    return torch.full((n,), value, dtype=torch.bfloat16, device=dev)


@dataclass
class LayerWeights:
    in_norm: torch.Tensor
    qkv: torch.Tensor      # [h_q + 2 h_kv, h]
    q_norm: torch.Tensor   # [d]
    k_norm: torch.Tensor   # [d]
    o: torch.Tensor        # [h, h_q]
    post_norm: torch.Tensor
    gate_up: torch.Tensor  # [2 h_ffn, h]
    down: torch.Tensor     # [h, h_ffn]


def _layer(cfg: ModelConfig, g, dev) -> LayerWeights:
    return LayerWeights(
        in_norm=_ones(cfg.h, dev), qkv=_normal((cfg.qkv_out, cfg.h), g, dev), q_norm=_ones(cfg.d, dev),
        k_norm=_ones(cfg.d, dev), o=_normal((cfg.h, cfg.h_q), g, dev), post_norm=_ones(cfg.h, dev),
        gate_up=_normal((2 * cfg.h_ffn, cfg.h), g, dev), down=_normal((cfg.h, cfg.h_ffn), g, dev))


@dataclass
class TargetWeights:
    emb: torch.Tensor       # [V, h]
    layers: list[LayerWeights]
    final_norm: torch.Tensor
    lm_head: torch.Tensor   # [V, h] (untied)

    @classmethod
    def random(cls, cfg: ModelConfig, seed: int, dev) -> "TargetWeights":
        g = torch.Generator(device=dev).manual_seed(seed)
        emb = _normal((cfg.V, cfg.h), g, dev)
        layers = [_layer(cfg, g, dev) for _ in range(cfg.L)]
        return cls(emb=emb, layers=layers, final_norm=_ones(cfg.h, dev), lm_head=_normal((cfg.V, cfg.h), g, dev))


@dataclass
class DrafterWeights:
    fc: torch.Tensor          # [h, n_feat * h]
    hidden_norm: torch.Tensor
    layers: list[LayerWeights]
    final_norm: torch.Tensor  # = logit_scale

    @classmethod
    def random(cls, cfg: ModelConfig, dcfg: DrafterConfig, n_feat: int, seed: int, dev) -> "DrafterWeights":
        g = torch.Generator(device=dev).manual_seed(seed + 7919)
        return cls(fc=_normal((cfg.h, n_feat * cfg.h), g, dev), hidden_norm=_ones(cfg.h, dev),
                   layers=[_layer(cfg, g, dev) for _ in range(dcfg.layers)],
                   final_norm=_ones(cfg.h, dev, dcfg.logit_scale))


def rope_inv_freq(cfg: ModelConfig, dev) -> torch.Tensor:
    """fp32 inv_freq[i] = theta^(-2i/d), i < d/2 (shared by kernels and the oracle)."""
    i = torch.arange(0, cfg.d, 2, dtype=torch.float64)
    return (1.0 / (cfg.rope_theta ** (i / cfg.d))).to(torch.float32).to(dev)
