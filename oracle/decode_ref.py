"""CPU restatement of one Qwen2 / Qwen2.5 / Qwen3 decode step -- TEST INFRASTRUCTURE.

This file is the *oracle* for the decode MegaKernel.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import it; the product path (``paper_2605_11581_b200``)
never does and fails loudly when its CUDA library is missing.

Provenance.  The reference at /root/reference has NO numeric decode path
(``SPEC.md:181``: "No numerical computation of operator outputs"); its only
statement of the step is the operator-kind list ``pkg/src/mkplan/graph_ir.py:48-56``
(RmsNorm, Gemm, AttentionQK, Softmax, AttentionPV, Swiglu, ResidualAdd, LmHead)
and ``PAPER.md:216-218``.  The arithmetic therefore follows the published
Qwen2/Qwen3 decoder definition (Hugging Face ``transformers`` 5.5.0,
``models/qwen2/modeling_qwen2.py`` and ``models/qwen3/modeling_qwen3.py``):

    x -> RMSNorm(eps) -> q,k,v = W x (+bias, Qwen2) [-> per-head RMSNorm on q,k, Qwen3]
      -> RoPE(theta, rotate-half) -> append k,v -> GQA softmax(q K^T / sqrt(d)) V
      -> W_o -> +x -> RMSNorm -> W_down(SiLU(W_gate x) * W_up x) -> +
    final RMSNorm -> LM head -> argmax.

Parity pin: ``tools/make_decode_golden.py`` runs ``transformers.Qwen2ForCausalLM`` /
``Qwen3ForCausalLM`` in the build container (fp32 compute on the same bf16-rounded
weights) and stores logits / tokens under ``tests/golden/decode_*.npz``;
``tests/test_oracle_decode.py`` checks this restatement against those fixtures.  Parity of the numeric half is pinned to Hugging Face, not to the
reference repo (which has nothing to pin against).

Numerical contract shared with the CUDA kernel: weights are bf16 in memory and
used exactly (upcast to fp32), all activations and accumulations are fp32, the
KV cache stores bf16 (``kv_dtype``), RoPE factors come from the fp32 table
``weights.rope_table``.
"""

from __future__ import annotations

import math

import torch


def _rmsnorm(x: torch.Tensor, gain: torch.Tensor, eps: float) -> torch.Tensor:
    # modeling_qwen2.Qwen2RMSNorm.forward: x * rsqrt(mean(x^2) + eps) * weight
    var = x.pow(2).mean(-1, keepdim=True)
    return x * torch.rsqrt(var + eps) * gain


def _rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """modeling_qwen2.apply_rotary_pos_emb with rotate_half.

    x: [..., heads, D]; cos/sin: [..., D/2] broadcast over heads."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    c, s = cos.unsqueeze(-2), sin.unsqueeze(-2)
    return torch.cat((x1 * c - x2 * s, x2 * c + x1 * s), dim=-1)


class RefDecoder:
    """Greedy decoder over fp32-upcast bf16 weights with an explicit KV cache."""

    def __init__(self, cfg, weights, max_ctx: int, cos: torch.Tensor, sin: torch.Tensor,
                 kv_dtype: torch.dtype = torch.bfloat16, batch: int = 1):
        self.cfg = cfg
        self.max_ctx = max_ctx
        self.kv_dtype = kv_dtype
        self.batch = batch
        self.cos = cos.float().cpu()
        self.sin = sin.float().cpu()
        f = lambda t: None if t is None else t.detach().to("cpu", torch.float32)
        self.embed = f(weights.embed)
        self.final_norm = f(weights.final_norm)
        self.lm_head = self.embed if weights.lm_head is None else f(weights.lm_head)
        self.layers = []
        for lw in weights.layers:
            wqkv = torch.cat([f(lw.wq), f(lw.wk), f(lw.wv)], 0)
            bqkv = None
            if lw.bq is not None:
                bqkv = torch.cat([f(lw.bq), f(lw.bk), f(lw.bv)], 0)
            self.layers.append(dict(
                ln1=f(lw.ln1), wqkv=wqkv, bqkv=bqkv, q_norm=f(lw.q_norm), k_norm=f(lw.k_norm),
                wo=f(lw.wo), ln2=f(lw.ln2), wgu=torch.cat([f(lw.wgate), f(lw.wup)], 0), wdown=f(lw.wdown),
            ))
        L, B = cfg.n_layers, batch
        self.k_cache = torch.zeros(L, B, cfg.n_kv_heads, max_ctx, cfg.head_dim, dtype=kv_dtype)
        self.v_cache = torch.zeros_like(self.k_cache)

    # -- one decode step for a batch of sequences (each at its own position) --
    @torch.no_grad()
    def step(self, tokens, positions) -> torch.Tensor:
        """tokens, positions: length-B int sequences.  Returns logits [B, V] fp32."""
        cfg = self.cfg
        tokens = torch.as_tensor(tokens, dtype=torch.long).reshape(-1)
        positions = torch.as_tensor(positions, dtype=torch.long).reshape(-1)
        B = tokens.numel()
        assert B <= self.batch
        D, G = cfg.head_dim, cfg.group
        scale = 1.0 / math.sqrt(D)
        h = self.embed[tokens]                                           # [B, H]
        cos, sin = self.cos[positions], self.sin[positions]              # [B, D/2]
        for l, w in enumerate(self.layers):
            x = _rmsnorm(h, w["ln1"], cfg.rms_eps)
            qkv = x @ w["wqkv"].T
            if w["bqkv"] is not None:
                qkv = qkv + w["bqkv"]
            q = qkv[:, :cfg.q_dim].reshape(B, cfg.n_q_heads, D)
            k = qkv[:, cfg.q_dim:cfg.q_dim + cfg.kv_dim].reshape(B, cfg.n_kv_heads, D)
            v = qkv[:, cfg.q_dim + cfg.kv_dim:].reshape(B, cfg.n_kv_heads, D)
            if w["q_norm"] is not None:                                   # Qwen3Attention
                q = _rmsnorm(q, w["q_norm"], cfg.rms_eps)
                k = _rmsnorm(k, w["k_norm"], cfg.rms_eps)
            q = _rope(q, cos, sin)
            k = _rope(k, cos, sin)
            attn = torch.empty(B, cfg.q_dim)
            for b in range(B):
                p = int(positions[b])
                self.k_cache[l, b, :, p] = k[b].to(self.kv_dtype)
                self.v_cache[l, b, :, p] = v[b].to(self.kv_dtype)
                K = self.k_cache[l, b, :, :p + 1].float()                 # [kv, T, D]
                V = self.v_cache[l, b, :, :p + 1].float()
                qb = (q[b] * scale).reshape(cfg.n_kv_heads, G, D)
                s = torch.einsum("hgd,htd->hgt", qb, K)
                pr = torch.softmax(s, dim=-1)
                attn[b] = torch.einsum("hgt,htd->hgd", pr, V).reshape(-1)
            h = h + attn @ w["wo"].T
            x = _rmsnorm(h, w["ln2"], cfg.rms_eps)
            gu = x @ w["wgu"].T
            g, u = gu[:, :cfg.intermediate], gu[:, cfg.intermediate:]
            act = g * torch.sigmoid(g) * u                                # SiLU(g) * u
            h = h + act @ w["wdown"].T
        hn = _rmsnorm(h, self.final_norm, cfg.rms_eps)
        return hn @ self.lm_head.T

    @torch.no_grad()
    def prefill(self, prompt, b: int = 0) -> torch.Tensor:
        """Causal pass over ``prompt`` for sequence ``b``; fills the KV cache and
        returns the last position's logits [V].  Token-parallel restatement of
        ``len(prompt)`` consecutive ``step`` calls."""
        cfg = self.cfg
        toks = torch.as_tensor(prompt, dtype=torch.long).reshape(-1)
        T = toks.numel()
        D, G = cfg.head_dim, cfg.group
        scale = 1.0 / math.sqrt(D)
        h = self.embed[toks]
        cos, sin = self.cos[:T], self.sin[:T]
        mask = torch.full((T, T), float("-inf")).triu(1)
        for l, w in enumerate(self.layers):
            x = _rmsnorm(h, w["ln1"], cfg.rms_eps)
            qkv = x @ w["wqkv"].T
            if w["bqkv"] is not None:
                qkv = qkv + w["bqkv"]
            q = qkv[:, :cfg.q_dim].reshape(T, cfg.n_q_heads, D)
            k = qkv[:, cfg.q_dim:cfg.q_dim + cfg.kv_dim].reshape(T, cfg.n_kv_heads, D)
            v = qkv[:, cfg.q_dim + cfg.kv_dim:].reshape(T, cfg.n_kv_heads, D)
            if w["q_norm"] is not None:
                q = _rmsnorm(q, w["q_norm"], cfg.rms_eps)
                k = _rmsnorm(k, w["k_norm"], cfg.rms_eps)
            q = _rope(q, cos, sin)
            k = _rope(k, cos, sin)
            self.k_cache[l, b, :, :T] = k.transpose(0, 1).to(self.kv_dtype)
            self.v_cache[l, b, :, :T] = v.transpose(0, 1).to(self.kv_dtype)
            K = self.k_cache[l, b, :, :T].float()
            V = self.v_cache[l, b, :, :T].float()
            qh = (q * scale).reshape(T, cfg.n_kv_heads, G, D)
            s = torch.einsum("thgd,hsd->hgts", qh, K) + mask
            pr = torch.softmax(s, dim=-1)
            attn = torch.einsum("hgts,hsd->thgd", pr, V).reshape(T, cfg.q_dim)
            h = h + attn @ w["wo"].T
            x = _rmsnorm(h, w["ln2"], cfg.rms_eps)
            gu = x @ w["wgu"].T
            g, u = gu[:, :cfg.intermediate], gu[:, cfg.intermediate:]
            h = h + (g * torch.sigmoid(g) * u) @ w["wdown"].T
        hn = _rmsnorm(h[-1:], self.final_norm, cfg.rms_eps)
        return (hn @ self.lm_head.T)[0]

    @torch.no_grad()
    def generate(self, prompt, max_new_tokens: int, stepwise_prefill: bool = False):
        """Greedy decode.  Returns (tokens, per-step logits list)."""
        prompt = [int(t) for t in prompt]
        if stepwise_prefill:
            logits = None
            for p, t in enumerate(prompt):
                logits = self.step([t], [p])[0]
        else:
            logits = self.prefill(prompt)
        out, all_logits = [], []
        pos = len(prompt)
        for _ in range(max_new_tokens):
            all_logits.append(logits)
            nxt = int(torch.argmax(logits))
            out.append(nxt)
            if len(out) == max_new_tokens:
                break
            logits = self.step([nxt], [pos])[0]
            pos += 1
        return out, all_logits
