"""Hybrid prefill/decode engine hook.

The paper's online half (``PAPER.md:239-250``) keeps the serving engine's own
operators for Prefill and switches to the MegaKernel plugin for Decode
("phase-adaptive execution").  The reference implements neither (``SPEC.md:8``
puts the engine out of scope), so this class defines the hook: ``generate``
runs a prefill backend to fill the KV cache the plugin owns, then enqueues one
persistent-kernel launch per generated token with the token / position state
resident on the device (no host round trip inside the decode loop).

Prefill backends.  ``"decode"`` (the only one built so far) feeds the prompt
through the decode kernel itself, one launch per prompt token -- correct, and
already ~0.7 ms per token, but not compute-efficient for long prompts.  The
tensor-core (tcgen05) prefill GEMM / attention kernels are SURVEY.md section
8(f) row 2; they plug in here by filling ``plugin.kv_view()`` and returning the
first decode token.  There is no CPU or PyTorch-op fallback on this path.
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
                 device: int = 0, prefill_backend: str = "decode"):
        if prefill_backend != "decode":
            raise NotImplementedError(f"prefill backend {prefill_backend!r} is not built (SURVEY.md 8(f).2)")
        self.cfg = cfg
        self.prefill_backend = prefill_backend
        self.plugin = MegaKernelPlugin(cfg, schedule or default_schedule(cfg), max_ctx=max_ctx, device=device)
        self.plugin.bind_weights(weights)

    def prefill(self, prompt_ids) -> None:
        """Fill the KV cache for ``prompt_ids[:-1]`` and leave the device state at the
        last prompt token, ready for the first decode launch."""
        plug = self.plugin
        prompt = torch.as_tensor(prompt_ids, dtype=torch.int32, device=plug.device)
        if prompt.numel() < 1:
            raise ValueError("empty prompt")
        if prompt.numel() + 1 > plug.max_ctx:
            raise ValueError("prompt does not fit the KV cache")
        for pos in range(prompt.numel() - 1):
            plug.tokens.copy_(prompt[pos:pos + 1])
            plug.positions.fill_(pos)
            plug.enqueue(want_logits=False, auto_advance=False)
        plug.tokens.copy_(prompt[-1:])
        plug.positions.fill_(prompt.numel() - 1)

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
