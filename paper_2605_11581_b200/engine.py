"""Hybrid prefill/decode engine hook.

The paper's online half (``PAPER.md:239-250``) keeps the serving engine's own
operators for Prefill and switches to the MegaKernel plugin for Decode
("phase-adaptive execution").  The reference implements neither (``SPEC.md:8``
puts the engine out of scope), so this class defines the hook: ``generate``
runs a prefill backend to fill the KV cache the plugin owns, then enqueues one
persistent-kernel launch per generated token with the token / position state
resident on the device (no host round trip inside the decode loop).

Prefill backends.  ``"decode"`` feeds the prompt through the decode kernel itself, one launch per prompt token --
bit-for-bit the decode path's cache, ~0.9 ms per token, not compute-efficient for long prompts.
``"library"`` is the paper's own arrangement (``PAPER.md:248``: Prefill stays on the serving engine's native
operators): library GEMMs (cuBLAS through ``torch.matmul``) and library attention fill the KV cache the plugin
owns, token-parallel; it is the BASELINE the hand-written tensor-core (tcgen05) prefill GEMM / attention kernels
of SURVEY.md section 8(f) row 2 have to beat, not a product kernel, and it is never used unless asked for.
``"tensor"`` (the default) is the hand-written replacement of that library path (``prefill.py``): a tcgen05 / tensor-memory GEMM
with fused bias / residual / SwiGLU epilogues, a tcgen05 causal flash-attention kernel (``csrc/prefill_attn.cu``) and
the row kernels around them.  ``prefill_planes`` = 1 (the default) feeds bf16 activations to the GEMMs -- the library
path's precision class at 0.7x its time (Qwen2.5-7B, 4096 tokens: 59 ms against 84 ms); 2 feeds each fp32 activation
as hi + lo bf16 planes (GEMMs exact to fp32, 1.6x the time) for callers that want the decode kernel's contract.
Every backend ends with the device state at the last prompt token, so the first generated token already comes
from a MegaKernel launch.  There is no CPU fallback on any path.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .model_config import ModelConfig
from .plugin import MegaKernelPlugin
from .schedules import default_schedule
from .task_table import KernelSchedule
from .weights import DecoderWeights


@dataclass
class GenerationResult:
    tokens: list
    prefill_launches: int
    decode_launches: int


class HybridEngine:
    """Prefill -> decode switch around one ``MegaKernelPlugin``."""

    def __init__(self, cfg: ModelConfig, weights: DecoderWeights, max_ctx: int, schedule: KernelSchedule | None = None,
                 device: int = 0, prefill_backend: str = "tensor", prefill_dtype: torch.dtype = torch.float32,
                 prefill_planes: int = 1, prefill_attention: str | None = None):
        if prefill_backend not in ("decode", "library", "tensor"):
            raise NotImplementedError(f"prefill backend {prefill_backend!r} does not exist")
        self.cfg = cfg
        self.prefill_backend = prefill_backend
        self.prefill_dtype = prefill_dtype
        self.plugin = MegaKernelPlugin(cfg, schedule or default_schedule(cfg), max_ctx=max_ctx, device=device)
        self.plugin.bind_weights(weights, keep_source=(prefill_backend == "library"))
        self._tensor_prefill = None
        if prefill_backend == "tensor":
            from .prefill import TensorCorePrefill

            self._tensor_prefill = TensorCorePrefill(cfg, weights, self.plugin, planes=prefill_planes, attention=prefill_attention)

    def prefill(self, prompt_ids) -> None:
        """Fill the KV cache for ``prompt_ids[:-1]`` and leave the device state at the
        last prompt token, ready for the first decode launch."""
        plug = self.plugin
        prompt = torch.as_tensor(prompt_ids, dtype=torch.int32, device=plug.device)
        if prompt.numel() < 1:
            raise ValueError("empty prompt")
        if prompt.numel() + 1 > plug.max_ctx:
            raise ValueError("prompt does not fit the KV cache")
        if self.prefill_backend in ("library", "tensor"):
            if self.prefill_backend == "library":
                self._library_prefill(prompt[:-1].long())
            else:
                self._tensor_prefill.run(prompt[:-1])
            plug.tokens.copy_(prompt[-1:])
            plug.positions.fill_(prompt.numel() - 1)
            return
        for pos in range(prompt.numel() - 1):
            plug.tokens.copy_(prompt[pos:pos + 1])
            plug.positions.fill_(pos)
            plug.enqueue(want_logits=False, auto_advance=False)
        plug.tokens.copy_(prompt[-1:])
        plug.positions.fill_(prompt.numel() - 1)

    @torch.no_grad()
    def _library_prefill(self, toks: torch.Tensor) -> None:
        """Token-parallel causal pass over ``toks`` with library GEMMs / attention (see the module docstring);
        writes K and V of every layer into the plugin's cache.  ``prefill_dtype`` float32 keeps the decode path's
        numerical contract (bf16 weights used exactly, fp32 activations); bfloat16 is the fast setting."""
        import torch.nn.functional as F

        cfg, plug, dt = self.cfg, self.plugin, self.prefill_dtype
        w = plug._weights
        T = toks.numel()
        if T == 0:
            return
        D, G = cfg.head_dim, cfg.group
        cos, sin = (t[:T].to(torch.float32) for t in plug._rope)
        kc, vc = plug.kv_view()

        def norm(x, gain):
            xf = x.float()
            return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + cfg.rms_eps) * gain.float()).to(dt)

        def rope(x):                       # [T, heads, D] fp32, rotate-half
            x1, x2 = x[..., :D // 2], x[..., D // 2:]
            c, s_ = cos[:, None, :], sin[:, None, :]
            return torch.cat((x1 * c - x2 * s_, x2 * c + x1 * s_), dim=-1)

        def lin(x, weight, bias=None):
            y = x @ weight.to(dt).T
            return y if bias is None else y + bias.to(dt)

        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            h = w.embed[toks].float()
            for l, lw in enumerate(w.layers):
                x = norm(h, lw.ln1)
                q = lin(x, lw.wq, lw.bq).float().reshape(T, cfg.n_q_heads, D)
                k = lin(x, lw.wk, lw.bk).float().reshape(T, cfg.n_kv_heads, D)
                v = lin(x, lw.wv, lw.bv).float().reshape(T, cfg.n_kv_heads, D)
                if lw.q_norm is not None:
                    q = norm(q, lw.q_norm).float()
                    k = norm(k, lw.k_norm).float()
                q, k = rope(q), rope(k)
                kb, vb = k.to(torch.bfloat16), v.to(torch.bfloat16)
                kc[l, 0, :, :T] = kb.transpose(0, 1)
                vc[l, 0, :, :T] = vb.transpose(0, 1)
                # attention over the bf16 cache contents, as the decode kernel sees them
                qh = q.transpose(0, 1).to(dt)[None]                                   # [1, nq, T, D]
                kh = kb.transpose(0, 1).to(dt).repeat_interleave(G, dim=0)[None]
                vh = vb.transpose(0, 1).to(dt).repeat_interleave(G, dim=0)[None]
                attn = F.scaled_dot_product_attention(qh, kh, vh, is_causal=True)[0].transpose(0, 1).reshape(T, cfg.q_dim)
                h = h + lin(attn, lw.wo).float()
                x = norm(h, lw.ln2)
                g_ = lin(x, lw.wgate).float()
                u = lin(x, lw.wup).float()
                h = h + lin((g_ * torch.sigmoid(g_) * u).to(dt), lw.wdown).float()
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev

    @torch.no_grad()
    def generate(self, prompt_ids, max_new_tokens: int) -> GenerationResult:
        plug = self.plugin
        n_prompt = len(prompt_ids)
        if n_prompt + max_new_tokens > plug.max_ctx:
            raise ValueError("prompt + max_new_tokens exceed the KV cache")
        start = plug.launches
        self.prefill(prompt_ids)
        prefill_launches = plug.launches - start
        out = torch.empty(max_new_tokens, dtype=torch.int32, device=plug.device)
        for i in range(max_new_tokens):
            plug.enqueue(want_logits=False, auto_advance=True)   # one launch per token, state stays on the device
            out[i:i + 1].copy_(plug.next_token)
        plug.check()
        return GenerationResult(out.cpu().tolist(), prefill_launches, plug.launches - start - prefill_launches)

    def close(self) -> None:
        self.plugin.close()
