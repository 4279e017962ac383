"""Tensor-parallel restatement of the CPU decode oracle -- TEST INFRASTRUCTURE.

Splits ``oracle/decode_ref.py``'s step the way the kernel's tensor-parallel ranks do (
Megatron-style): rank r owns a slice of the q/kv heads, of the MLP intermediate channels and of the
vocabulary (``DecoderWeights.shard``); attention and the MLP each end in a partial sum over the hidden
size that is added across ranks in rank order, rank 0's partial carrying the residual -- exactly the
slots ``csrc/adamk.cu`` publishes through peer memory.  Used by the CPU tests (single process and
world-size-2 gloo) to show that the sharding is equivalent to the unsharded oracle; the reference has no
parallelism of any kind, so there is nothing of its own to pin against.
"""

from __future__ import annotations

import torch

from .decode_ref import RefDecoder, _rmsnorm


class RankRef(RefDecoder):
    """One tensor-parallel rank: a RefDecoder over the rank's weight shard whose ``*_partial`` methods
    return the rank's contribution to the hidden state."""

    def __init__(self, full_cfg, weights, rank: int, tp: int, max_ctx: int, cos, sin):
        super().__init__(full_cfg.shard(tp), weights.shard(rank, tp), max_ctx, cos, sin)
        self.rank, self.tp, self.full_cfg = rank, tp, full_cfg
        f = lambda t: t.detach().to("cpu", torch.float32)
        self.embed = f(weights.embed)                      # whole table: every rank gathers the input row
        self.lm_head = f(weights.shard(rank, tp).lm_head)  # the rank's vocabulary slice

    @torch.no_grad()
    def attn_partial(self, l: int, h: torch.Tensor, pos: int) -> torch.Tensor:
        """W_o[:, heads_r] . attention_r(h) for one sequence at position ``pos`` (appends K/V)."""
        import math
        cfg, w = self.cfg, self.layers[l]
        D, G = cfg.head_dim, cfg.group
        x = _rmsnorm(h, w["ln1"], cfg.rms_eps)
        qkv = x @ w["wqkv"].T
        if w["bqkv"] is not None:
            qkv = qkv + w["bqkv"]
        q = qkv[:cfg.q_dim].reshape(cfg.n_q_heads, D)
        k = qkv[cfg.q_dim:cfg.q_dim + cfg.kv_dim].reshape(cfg.n_kv_heads, D)
        v = qkv[cfg.q_dim + cfg.kv_dim:].reshape(cfg.n_kv_heads, D)
        if w["q_norm"] is not None:
            q = _rmsnorm(q, w["q_norm"], cfg.rms_eps)
            k = _rmsnorm(k, w["k_norm"], cfg.rms_eps)
        from .decode_ref import _rope
        cos, sin = self.cos[pos], self.sin[pos]
        q, k = _rope(q, cos, sin), _rope(k, cos, sin)
        self.k_cache[l, 0, :, pos] = k.to(self.kv_dtype)
        self.v_cache[l, 0, :, pos] = v.to(self.kv_dtype)
        K = self.k_cache[l, 0, :, :pos + 1].float()
        V = self.v_cache[l, 0, :, :pos + 1].float()
        qb = (q / math.sqrt(D)).reshape(cfg.n_kv_heads, G, D)
        pr = torch.softmax(torch.einsum("hgd,htd->hgt", qb, K), dim=-1)
        attn = torch.einsum("hgt,htd->hgd", pr, V).reshape(-1)
        return attn @ w["wo"].T

    @torch.no_grad()
    def mlp_partial(self, l: int, h: torch.Tensor) -> torch.Tensor:
        cfg, w = self.cfg, self.layers[l]
        x = _rmsnorm(h, w["ln2"], cfg.rms_eps)
        gu = x @ w["wgu"].T
        g, u = gu[:cfg.intermediate], gu[cfg.intermediate:]
        return (g * torch.sigmoid(g) * u) @ w["wdown"].T

    @torch.no_grad()
    def logits_slice(self, h: torch.Tensor) -> torch.Tensor:
        return _rmsnorm(h, self.final_norm, self.cfg.rms_eps) @ self.lm_head.T


def tp_step(ranks: list[RankRef], token: int, pos: int, reduce=None) -> torch.Tensor:
    """One decode step over ``ranks`` (all of them in one process, or just the local one with ``reduce`` an
    all-reduce over processes).  Partials are summed in rank order with the residual first, as the kernel's
    slot gather does.  Returns the concatenated (or local-slice) logits."""
    h = ranks[0].embed[token]
    n_layers = ranks[0].cfg.n_layers
    for l in range(n_layers):
        parts = [r.attn_partial(l, h, pos) for r in ranks]
        h = h + (reduce(parts[0]) if reduce else sum(parts[1:], parts[0]))
        parts = [r.mlp_partial(l, h) for r in ranks]
        h = h + (reduce(parts[0]) if reduce else sum(parts[1:], parts[0]))
    return torch.cat([r.logits_slice(h) for r in ranks])
