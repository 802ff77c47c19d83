"""Model shapes of the benchmark configurations (BASELINE.json configs)."""

from __future__ import annotations

from dataclasses import dataclass, field

from ..cost_model import CostModelParams


@dataclass(frozen=True)
class ModelConfig:
    """Qwen3-style decoder: RMSNorm, GQA with per-head q/k norm, RoPE, SwiGLU, untied LM head."""

    name: str
    L: int
    h: int
    n_q: int
    n_kv: int
    d: int
    h_ffn: int
    V: int
    rope_theta: float = 1.0e6
    eps: float = 1.0e-6

    @property
    def h_q(self) -> int:
        return self.n_q * self.d

    @property
    def h_kv(self) -> int:
        return self.n_kv * self.d

    @property
    def qkv_out(self) -> int:
        return self.h_q + 2 * self.h_kv

    def cost_params(self, peak_flops: float, bandwidth: float) -> CostModelParams:
        """Appendix-D profile of this model (cost_model.py:26-57) at the given peaks."""
        return CostModelParams(L=self.L, h=self.h, n_q=self.n_q, n_kv=self.n_kv, d=self.d, h_ffn=self.h_ffn,
                               V=self.V, bp=2, peak_flops=peak_flops, bandwidth=bandwidth)


@dataclass(frozen=True)
class DrafterConfig:
    """DFlash-style block drafter (block 16 at PAPER.md:332).

    ``layers`` Qwen3 decoder layers of the target width; target hidden states of
    ``feat_layers`` are concatenated, projected by ``fc`` + ``hidden_norm`` and
    injected as per-layer context K/V; queries are [bonus] + gamma mask tokens,
    attention is non-causal, logits are read at the gamma mask positions.
    ``logit_scale`` multiplies the drafter's final-norm weight — the documented
    knob that makes random-init drafter rows peaked enough for non-trivial
    adaptive trees.
    """

    layers: int = 5
    gamma: int = 16
    feat_layers: tuple[int, ...] = field(default=())
    mask_token: int = -1  # -1 -> V - 1
    logit_scale: float = 6.0


QWEN3_8B = ModelConfig("qwen3-8b", L=36, h=4096, n_q=32, n_kv=8, d=128, h_ffn=12288, V=151936)
QWEN3_32B = ModelConfig("qwen3-32b", L=64, h=5120, n_q=64, n_kv=8, d=128, h_ffn=25600, V=151936)
# Config 1 (CPU-runnable oracle): tiny but with the kernels' fixed head_dim of 128.
TINY = ModelConfig("tiny", L=2, h=256, n_q=4, n_kv=2, d=128, h_ffn=512, V=1024)

MODELS = {m.name: m for m in (QWEN3_8B, QWEN3_32B, TINY)}


def default_feat_layers(L: int, n: int = 5) -> tuple[int, ...]:
    """n target layers spread over [1, L-3] (DFlash-style feature taps)."""
    if L <= 2:
        return tuple(range(L))
    lo, hi = 1, max(1, L - 3)
    n = min(n, hi - lo + 1)
    return tuple(sorted({round(lo + i * (hi - lo) / max(1, n - 1)) for i in range(n)}))
