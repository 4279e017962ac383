"""Batched decode on the tensor cores (BASELINE.json configs[2]).

The MegaKernel streams the weights once per token of ONE sequence (GEMV on the CUDA cores); with ``B`` sequences in
flight the same weight bytes can serve all of them if the projections become ``[B, K] x [K, N]`` GEMMs.  This module
runs one decode step of ``B`` sequences with the operators of ``include/adamk_prefill.h``:

* projections (QKV, O, gate/up, down, LM head): the tcgen05 GEMM of ``csrc/prefill_gemm.cu`` with ``T = B`` (TMA
  zero-fills the unused token rows of the 128-row tile; the tensor work is free, the kernel is bound by streaming
  ``W``).  A decode-sized GEMM has fewer tiles than SMs, so K is split across SMs with an fp32-atomic epilogue
  (``EPI_ATOMIC``), which is what lets every SM pull weight bytes, and both activation planes ride in the one token
  tile, so a weight byte is read once.  SwiGLU is a row kernel on the gate/up result.
* activations enter the tensor cores as bf16 planes whose sum is the fp32 value -- three (hi + mid + lo, exact to
  fp32) while 3 B <= 128 rows still fit the one token tile, two (2^-17) beyond -- so the step keeps the MegaKernel's
  numerical contract (fp32 activations against exact bf16 weights) at no cost in time.
* ``adamk_batch_rope_store`` (per-sequence positions), ``adamk_batch_attention`` (split over 64-row chunks of
  each sequence's cache + merge) and ``adamk_batch_argmax`` (greedy pick, tokens / positions advanced on the device).

A step is 10 launches per layer; ``capture()`` records it once into a CUDA graph, after which a step is one graph
launch with no host work.  Prompts are filled by ``TensorCorePrefill`` into the same cache.  No CPU path.
"""

from __future__ import annotations

import ctypes as C

import torch

from .model_config import ModelConfig
from .plugin import AdamkError
from .prefill import (EPI_ATOMIC, GU_BLOCK, TensorCorePrefill, _lib, _ok, _ptr, _stream, gemm,
                      interleave_gate_up)
from .weights import DecoderWeights, rope_table


class _SequenceCache:
    """What ``TensorCorePrefill`` needs from a plugin, for one sequence of a ``BatchedDecoder``."""

    def __init__(self, owner: "BatchedDecoder", b: int):
        self.device, self.max_ctx, self._rope = owner.device, owner.max_ctx, owner._rope
        self._k, self._v = owner.k_cache[:, b:b + 1], owner.v_cache[:, b:b + 1]

    def kv_view(self):
        return self._k, self._v


class BatchedDecoder:
    def __init__(self, cfg: ModelConfig, weights: DecoderWeights, batch: int, max_ctx: int, device: int = 0, planes: int | None = None,
                 pdl: int = 2, l2_prefetch: bool = False):
        if not torch.cuda.is_available():
            raise AdamkError(-102, "no CUDA device: batched decode has no CPU fallback")
        if not 1 <= batch <= 128:
            raise ValueError("batch must be 1..128 (one 128-row GEMM tile)")
        if planes is None:      # three planes (activations exact to fp32) while they still share one 128-row token tile
            planes = 3 if 3 * batch <= 128 else 2
        if planes not in (1, 2, 3):
            raise ValueError("planes must be 1, 2 or 3")
        if cfg.vocab % 8 or cfg.hidden % 8 or cfg.intermediate % 8 or cfg.head_dim not in (64, 128):
            raise ValueError("batched decode needs vocab / hidden / intermediate sizes that are multiples of 8 and head_dim 64 or 128")
        self.lib = _lib()
        self.cfg, self.batch, self.max_ctx, self.planes = cfg, batch, int(max_ctx), planes
        # every GEMM pulls the next GEMM's weight into L2 while it waits for its own (measured: -3.6 % step time on
        # Qwen2.5-1.5B at batch 8, +9 % on Qwen2.5-7B whose GEMMs are already bandwidth-bound; off by default)
        self.l2_prefetch = bool(l2_prefetch)
        # programmatic dependent launch between the step's kernels (adamk_prefill_set_pdl): 1 = prologues overlap the previous
        # kernel's tail (-3.6 % step time at batch 8), 2 = also the first ring pass of every GEMM's weights issued ahead of
        # griddepcontrol.wait (-6.6 % at batch 8, -5 % at 16, +-0 at 64; profiles/r02_batch_pdl_ab.txt)
        self.pdl = int(pdl)
        dev = self.device = torch.device("cuda", device)
        cos, sin = rope_table(cfg, max_ctx)
        self._rope = (cos.to(dev), sin.to(dev))
        self._weights = weights
        self.embed = weights.embed.to(dev)
        self.final_norm = weights.final_norm.to(dev)
        self.lm_head = weights.lm_head_matrix.to(dev).contiguous()
        self.layers = []
        for lw in weights.layers:
            wgu = interleave_gate_up(lw.wgate.to(dev), lw.wup.to(dev))
            i_pad = wgu.shape[0] // 2
            wdown = lw.wdown.to(dev)
            if i_pad != cfg.intermediate:
                wdown = torch.nn.functional.pad(wdown, (0, i_pad - cfg.intermediate))
            self.layers.append(dict(
                ln1=lw.ln1.to(dev), ln2=lw.ln2.to(dev), wqkv=torch.cat((lw.wq, lw.wk, lw.wv), dim=0).to(dev).contiguous(),
                bqkv=None if lw.bq is None else torch.cat((lw.bq, lw.bk, lw.bv)).to(dev).float().contiguous(),
                wo=lw.wo.to(dev).contiguous(), wgu=wgu, wdown=wdown.contiguous(), i_pad=i_pad,
                q_norm=None if lw.q_norm is None else lw.q_norm.to(dev), k_norm=None if lw.k_norm is None else lw.k_norm.to(dev)))
        B, P, H, D, nq, nkv = batch, planes, cfg.hidden, cfg.head_dim, cfg.n_q_heads, cfg.n_kv_heads
        bf, f32 = torch.bfloat16, torch.float32
        self.k_cache = torch.zeros(cfg.n_layers, B, nkv, max_ctx, D, dtype=bf, device=dev)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.tokens = torch.zeros(B, dtype=torch.int32, device=dev)
        self.positions = torch.zeros(B, dtype=torch.int32, device=dev)
        self.next_token = torch.zeros(B, dtype=torch.int32, device=dev)
        self.h = torch.empty(B, H, dtype=f32, device=dev)
        self.xp = torch.empty(P, B, H, dtype=bf, device=dev)
        n_qkv, i_pad = (nq + 2 * nkv) * D, self.layers[0]["i_pad"]
        self.acc = torch.empty(B * (n_qkv + 2 * i_pad), dtype=f32, device=dev)     # the two atomic GEMM targets, cleared together
        self.qkv = self.acc[:B * n_qkv].view(B, n_qkv)
        self.gu = self.acc[B * n_qkv:].view(B, 2 * i_pad)
        self.q = torch.empty(nq, B, D, dtype=f32, device=dev)
        self.ap = torch.empty(P, B, nq * D, dtype=bf, device=dev)
        self.act = torch.empty(P, B, self.layers[0]["i_pad"], dtype=bf, device=dev)
        self.logits = torch.empty(B, cfg.vocab, dtype=f32, device=dev)
        ws = self.lib.adamk_batch_attention_workspace(B, nq, D, max_ctx)
        self.attn_ws = torch.empty(ws // 4, dtype=f32, device=dev)
        self.argmax_ws = torch.zeros(self.lib.adamk_batch_argmax_workspace(B), dtype=torch.uint8, device=dev)   # zero once; the kernel re-arms it
        self._graph = None
        self.launches_per_step = 0
        self.steps = 0
        # Host-side bound on the largest device position: positions advance on the device (argmax kernel, graph replay), so
        # the host counts auto-advancing steps since the last state it set and refuses the step that would leave the cache.
        # The kernels also guard themselves (a sequence past max_ctx writes nothing and attends inside the cache).
        self._pos_bound = 0

    # ---- prompts ----
    def prefill(self, b: int, prompt_ids) -> None:
        """Fill sequence ``b``'s cache from ``prompt_ids[:-1]`` and leave its state at the last prompt token."""
        prompt = torch.as_tensor(prompt_ids, dtype=torch.int32, device=self.device)
        if prompt.numel() < 1 or prompt.numel() + 1 > self.max_ctx:
            raise ValueError("prompt is empty or does not fit the KV cache")
        if prompt.numel() > 1:
            TensorCorePrefill(self.cfg, self._weights, _SequenceCache(self, b), planes=min(self.planes, 2),
                              layers=self.layers, embed=self.embed).run(prompt[:-1])
        if int(prompt.min()) < 0 or int(prompt.max()) >= self.cfg.vocab:
            raise ValueError("prompt holds token ids outside the vocabulary")
        self.tokens[b] = prompt[-1]
        self.positions[b] = prompt.numel() - 1
        self._pos_bound = max(self._pos_bound, prompt.numel() - 1)

    def set_state(self, tokens, positions) -> None:
        tok = torch.as_tensor(tokens, dtype=torch.int32).cpu()
        pos = torch.as_tensor(positions, dtype=torch.int32).cpu()
        if tok.numel() != self.batch or pos.numel() != self.batch:
            raise ValueError("set_state needs one token and one position per sequence")
        if int(tok.min()) < 0 or int(tok.max()) >= self.cfg.vocab:
            raise ValueError("token id outside the vocabulary")
        if int(pos.min()) < 0 or int(pos.max()) >= self.max_ctx:
            raise ValueError(f"position outside the KV cache (max_ctx {self.max_ctx})")
        self.tokens.copy_(tok)
        self.positions.copy_(pos)
        self._pos_bound = int(pos.max())

    # ---- one step ----
    @torch.no_grad()
    def _enqueue(self, auto_advance: bool) -> int:
        self.lib.adamk_prefill_set_pdl(int(self.pdl))
        try:
            return self._enqueue_step(auto_advance)
        finally:
            self.lib.adamk_prefill_set_pdl(0)

    def _enqueue_step(self, auto_advance: bool) -> int:
        cfg, lib, st, B, P = self.cfg, self.lib, _stream(), self.batch, self.planes
        H, D, nq, nkv = cfg.hidden, cfg.head_dim, cfg.n_q_heads, cfg.n_kv_heads
        seq_stride = nkv * self.max_ctx * D
        cos, sin = self._rope
        n = 0
        _ok(lib.adamk_batch_embed(_ptr(self.tokens), B, _ptr(self.embed), H, cfg.vocab, _ptr(self.h), st))
        pf = self.l2_prefetch
        for l, lw in enumerate(self.layers):
            nxt = self.layers[l + 1]["wqkv"] if l + 1 < len(self.layers) else self.lm_head
            _ok(lib.adamk_batch_rmsnorm_split(_ptr(self.h), _ptr(lw["ln1"]), cfg.rms_eps, B, H, _ptr(self.xp), P,
                                              _ptr(self.acc), self.acc.numel(), st))
            gemm(self.xp, lw["wqkv"], self.qkv, bias=lw["bqkv"], epilogue=EPI_ATOMIC, prefetch=lw["wo"] if pf else None)
            _ok(lib.adamk_batch_rope_store(_ptr(self.qkv), B, nq, nkv, D, _ptr(lw["q_norm"]), _ptr(lw["k_norm"]), cfg.rms_eps,
                                           _ptr(cos), _ptr(sin), _ptr(self.positions), seq_stride, self.max_ctx, _ptr(self.q),
                                           _ptr(self.k_cache[l]), _ptr(self.v_cache[l]), st))
            _ok(lib.adamk_batch_attention(_ptr(self.q), _ptr(self.k_cache[l]), _ptr(self.v_cache[l]), _ptr(self.positions), B, nq,
                                          nkv, D, self.max_ctx, seq_stride, _ptr(self.attn_ws), _ptr(self.ap), P, st))
            gemm(self.ap, lw["wo"], self.h, epilogue=EPI_ATOMIC, prefetch=lw["wgu"] if pf else None)   # h += attn . Wo^T
            _ok(lib.adamk_prefill_rmsnorm_split(_ptr(self.h), _ptr(lw["ln2"]), cfg.rms_eps, B, H, _ptr(self.xp), P, st))
            gemm(self.xp, lw["wgu"], self.gu, epilogue=EPI_ATOMIC, prefetch=lw["wdown"] if pf else None)
            _ok(lib.adamk_batch_swiglu_split(_ptr(self.gu), B, lw["i_pad"], GU_BLOCK, _ptr(self.act), P, st))
            gemm(self.act, lw["wdown"], self.h, epilogue=EPI_ATOMIC, prefetch=nxt if pf else None)      # h += act . Wdown^T
            n += 10         # own kernels (attention is two)
        # LM head: also through the atomic epilogue (planes stacked, the 0.47 GB matrix is read once)
        _ok(lib.adamk_batch_rmsnorm_split(_ptr(self.h), _ptr(self.final_norm), cfg.rms_eps, B, H, _ptr(self.xp), P,
                                          _ptr(self.logits), self.logits.numel(), st))
        gemm(self.xp, self.lm_head, self.logits, epilogue=EPI_ATOMIC)
        adv = auto_advance
        _ok(lib.adamk_batch_argmax_sliced(_ptr(self.logits), B, cfg.vocab, _ptr(self.argmax_ws), _ptr(self.next_token),
                                          _ptr(self.tokens) if adv else None, _ptr(self.positions) if adv else None, st))
        return n + 4

    def capture(self) -> None:
        """Record one auto-advancing step into a CUDA graph (after a warm-up step on a side stream)."""
        tok, pos = self.tokens.clone(), self.positions.clone()
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self._enqueue(auto_advance=False)
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.launches_per_step = self._enqueue(auto_advance=True)
        self._graph = graph
        self.tokens.copy_(tok)
        self.positions.copy_(pos)

    def step(self, auto_advance: bool = True) -> torch.Tensor:
        """One decode step of all sequences; returns the device tensor of greedy tokens (int32 [B])."""
        if self._pos_bound >= self.max_ctx:
            raise AdamkError(-103, f"a sequence has reached max_ctx ({self.max_ctx}): the step would write past its KV cache")
        if auto_advance:
            self._pos_bound += 1
        if self._graph is not None and auto_advance:
            self._graph.replay()
        else:
            self.launches_per_step = self._enqueue(auto_advance)
        self.steps += 1
        return self.next_token
