"""CPU ORACLE — test infrastructure only, never the product path.

torch fp32 restatement of the Qwen3-style target and the DFlash-style block
drafter the engine runs on the GPU (paper_2605_29727_b200/engine).  The
reference package has no model at all ("No tensors are involved",
verify_sim.py:3-5), so this model arithmetic is "parity unpinned" against the
reference; it pins the GPU kernels to a plain dense implementation instead:
full (T x T) masked attention, no KV cache, no paging, no stream-K.

bf16 rounding happens at exactly the boundaries where the kernels store bf16
(normed activations, q/k/v after norm+RoPE, attention output, SwiGLU output);
everything else is fp32, so GPU vs oracle differ only by accumulation order.
"""

from __future__ import annotations

import torch


def bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def rope(x: torch.Tensor, pos: torch.Tensor, inv_freq: torch.Tensor) -> torch.Tensor:
    """rotate_half RoPE on [..., T, heads, 128] with fp32 angles pos * inv_freq."""
    ang = pos.to(torch.float32)[:, None] * inv_freq[None, :]  # [T, 64]
    cos = torch.cat([ang.cos(), ang.cos()], -1)[:, None, :]
    sin = torch.cat([ang.sin(), ang.sin()], -1)[:, None, :]
    x1, x2 = x[..., :64], x[..., 64:]
    rot = torch.cat([-x2, x1], -1)
    return x * cos + rot * sin


class RefModel:
    """Holds fp32 CPU copies of the engine's bf16 weights."""

    def __init__(self, cfg, tw, dw=None, feat_layers=(), inv_freq=None, device="cpu"):
        f = lambda t: t.detach().to(device, torch.float32)  # noqa: E731
        self.cfg, self.device = cfg, torch.device(device)
        self.emb, self.final_norm, self.lm_head = f(tw.emb), f(tw.final_norm), f(tw.lm_head)
        self.layers = [{k: f(getattr(lw, k)) for k in lw.__dataclass_fields__} for lw in tw.layers]
        self.feat_layers = tuple(feat_layers)
        self.inv_freq = f(inv_freq)
        if dw is not None:
            self.fc, self.hidden_norm, self.d_final = f(dw.fc), f(dw.hidden_norm), f(dw.final_norm)
            self.d_layers = [{k: f(getattr(lw, k)) for k in lw.__dataclass_fields__} for lw in dw.layers]

    # ------------------------------------------------------------ one layer
    def _attn_block(self, lw, x_in, pos, kv_x, kv_pos, mask, cfg):
        """q from x_in rows, k/v from kv_x rows; mask [Tq, Tk] bool."""
        d, nq, nkv = cfg.d, cfg.n_q, cfg.n_kv
        qkv_q = x_in @ lw["qkv"].t()
        qkv_k = kv_x @ lw["qkv"].t()
        q = qkv_q[:, : nq * d].view(-1, nq, d)
        k = qkv_k[:, nq * d: (nq + nkv) * d].view(-1, nkv, d)
        v = qkv_k[:, (nq + nkv) * d:].view(-1, nkv, d)
        q = bf(rope(rmsnorm(q, lw["q_norm"], cfg.eps), pos, self.inv_freq))
        k = bf(rope(rmsnorm(k, lw["k_norm"], cfg.eps), kv_pos, self.inv_freq))
        v = bf(v)
        g = nq // nkv
        k = k.repeat_interleave(g, dim=1)
        v = v.repeat_interleave(g, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, k) / (d ** 0.5)
        s = s.masked_fill(~mask[None], float("-inf"))
        p = torch.softmax(s, -1)
        o = torch.einsum("hqk,khd->qhd", p, v).reshape(-1, nq * d)
        return bf(o) @ lw["o"].t()

    def _mlp(self, lw, x):
        gu = x @ lw["gate_up"].t()
        f = gu.shape[-1] // 2
        gt, up = gu[:, :f], gu[:, f:]
        act = bf(gt / (1 + torch.exp(-gt)) * up)
        return act @ lw["down"].t()

    # --------------------------------------------------------------- target
    def target(self, tokens, pos, mask):
        """Dense target forward: tokens/pos [T], mask [T, T] -> (logits fp32 [T, V], features [T, n_feat*h])."""
        cfg = self.cfg
        tokens = torch.as_tensor(tokens, dtype=torch.long, device=self.device)
        pos = torch.as_tensor(pos, device=self.device)
        mask = mask.to(self.device)
        resid = self.emb[tokens].clone()
        feats = []
        for li, lw in enumerate(self.layers):
            x = bf(rmsnorm(resid, lw["in_norm"], cfg.eps))
            resid = resid + self._attn_block(lw, x, pos, x, pos, mask, cfg)
            x = bf(rmsnorm(resid, lw["post_norm"], cfg.eps))
            resid = resid + self._mlp(lw, x)
            if li in self.feat_layers:
                feats.append(bf(resid))
        x = bf(rmsnorm(resid, self.final_norm, cfg.eps))
        feat = torch.cat(feats, -1) if feats else None
        return x @ self.lm_head.t(), feat

    # -------------------------------------------------------------- drafter
    def drafter(self, ctx_feat, c, bonus, gamma, mask_token):
        """Block drafter at context c: ctx_feat [c, n_feat*h] (target features of positions 0..c-1).

        Queries: [bonus, mask x gamma] at positions c..c+gamma; keys: context rows
        (positions 0..c-1, K/V from fc+hidden_norm features) + the block rows;
        non-causal.  Returns logits [gamma, V] of the mask positions.
        """
        cfg = self.cfg
        x_ctx = bf(rmsnorm(ctx_feat.to(self.device) @ self.fc.t(), self.hidden_norm, cfg.eps)) if c > 0 else None
        dev = self.device
        toks = torch.tensor([bonus] + [mask_token] * gamma, device=dev)
        bpos = torch.arange(c, c + gamma + 1, device=dev)
        cpos = torch.arange(0, c, device=dev)
        resid = self.emb[toks].clone()
        B = gamma + 1
        for li, lw in enumerate(self.d_layers):
            x = bf(rmsnorm(resid, lw["in_norm"], cfg.eps))
            kv_x = torch.cat([x_ctx, x]) if x_ctx is not None else x
            kv_pos = torch.cat([cpos, bpos])
            mask = torch.ones(B, kv_x.shape[0], dtype=torch.bool, device=dev)
            resid = resid + self._attn_block(lw, x, bpos, kv_x, kv_pos, mask, cfg)
            x = bf(rmsnorm(resid, lw["post_norm"], cfg.eps))
            resid = resid + self._mlp(lw, x)
        x = bf(rmsnorm(resid, self.d_final, cfg.eps))
        return (x @ self.lm_head.t())[1:]


def causal_mask(n: int) -> torch.Tensor:
    return torch.tril(torch.ones(n, n, dtype=torch.bool))


def verify_mask(c: int, anc: torch.Tensor) -> torch.Tensor:
    """Rows/cols: c committed positions (causal) then the t tree rows (prefix + ancestors)."""
    t = anc.shape[0]
    m = torch.zeros(c + t, c + t, dtype=torch.bool)
    m[:c, :c] = causal_mask(c)
    m[c:, :c] = True
    m[c:, c:] = anc
    return m


class RefPlugin:
    """The reference plugin protocol (sp/verify_sim.py:125-126,158-169) over :class:`RefModel`:
    fp64 drafter rows and greedy target tokens of the oracle model, for decoding config 1
    end to end on the CPU with ``specplan_port.decode_loop``.

    Alignment (SURVEY §8a′): with committed stream ``prefix``, the model sees
    ``prompt + prefix``; its last token is the pending root, the drafter's context is
    every earlier position.  ``near_ties`` collects the decisions whose fp32 margin is
    below ``tol`` x the row's max |logit| (top-2 target logits; the K-th/(K+1)-th drafter
    logits of a row): a GPU run may legitimately decide those differently (bf16 storage,
    fp32 sums in another order), no other.  A drafter near-tie can only change that
    cycle's tree; a target near-tie can change the committed stream.
    """

    def __init__(self, ref: RefModel, prompt, gamma: int, mask_token: int, top_k: int, tol: float = 2e-2):
        self.ref, self.prompt = ref, [int(t) for t in prompt]
        self.gamma, self.mask_token, self.top_k, self.tol = gamma, mask_token, top_k, tol
        self.near_ties: list[tuple[str, int]] = []  # (kind, committed length)
        self.target_gap: dict[int, float] = {}      # committed index -> top-2 gap / max|logit|
        self.drafter_gap: dict[int, float] = {}     # committed length -> min K/K+1 gap / max|logit|

    def drafter_marginals(self, prefix):
        full = self.prompt + [int(t) for t in prefix]
        c = len(full) - 1
        _, feat = self.ref.target(full[:-1], list(range(c)), causal_mask(c))
        lg = self.ref.drafter(feat, c, full[-1], self.gamma, self.mask_token)
        top = lg.topk(self.top_k + 1, dim=-1).values
        scale = lg.abs().amax(-1)
        self.drafter_gap[len(prefix)] = float(((top[:, self.top_k - 1] - top[:, self.top_k]) / scale).min())
        if bool(((top[:, self.top_k - 1] - top[:, self.top_k]) < self.tol * scale).any()):
            self.near_ties.append(("drafter", len(prefix)))
        return torch.softmax(lg.double(), -1).cpu().numpy()

    def next_token(self, seq, temperature: float = 0.0) -> int:
        if temperature != 0.0:
            raise ValueError("the oracle plugin decodes greedily")
        full = self.prompt + [int(t) for t in seq]
        n = len(full)
        lg, _ = self.ref.target(full, list(range(n)), causal_mask(n))
        top = lg[-1].topk(2).values
        self.target_gap[len(seq)] = float(top[0] - top[1]) / float(lg[-1].abs().max())
        if float(top[0] - top[1]) < self.tol * float(lg[-1].abs().max()):
            self.near_ties.append(("target", len(seq)))
        return int(torch.argmax(lg[-1]))  # first max on ties, as np.argmax (sp/verify_sim.py:107-109)
