"""W4A16 (GPTQ-format) weights for the decode MegaKernel.

The paper evaluates GPTQ-W4A16 checkpoints (``PAPER.md:252-261,312-313``); the reference models them as 4-bit codes plus
one two-byte scale per group of 128 reduction elements (``pkg/src/mkplan/graph_ir.py:296-318``: ``packed = n * k / 2``,
``scales = n * ceil(k / 128) * 2`` bytes).  This module holds that container and a round-to-nearest quantiser that
produces it from bf16 weights (there is no network for real GPTQ checkpoints; the calibration that GPTQ adds changes
which codes are chosen, not the format or the kernel).  ``W[n][k] = (q[n][k] - 8) * s[n][k // 128]``.

The kernel never dequantises on the host: ``MegaKernelPlugin.bind_weights`` hands the codes and scales to the device
packer (``adamk_bind_weights_w4a16``).  The reference dequantisation used by the tests lives in ``oracle/w4a16_ref.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .weights import DecoderWeights

GROUP = 128
MATRICES = ("wq", "wk", "wv", "wo", "wgate", "wup", "wdown")


@dataclass
class QuantMatrix:
    q: torch.Tensor   # uint8 [N, K / 2]: element k of a row in byte k // 2, even k in the low nibble
    s: torch.Tensor   # float16 [N, ceil(K / 128)]

    @property
    def shape(self) -> tuple[int, int]:
        return self.q.shape[0], self.q.shape[1] * 2

    def to(self, device) -> "QuantMatrix":
        return QuantMatrix(self.q.to(device).contiguous(), self.s.to(device).contiguous())

    def nbytes(self) -> int:
        return self.q.numel() + self.s.numel() * 2


def quantize_matrix(w: torch.Tensor) -> QuantMatrix:
    """Symmetric round-to-nearest 4-bit codes with one fp16 scale per (row, group of 128)."""
    n, k = w.shape
    if k % 8:
        raise ValueError("K must be a multiple of 8")
    wf = w.detach().float().cpu()
    ng = -(-k // GROUP)
    pad = ng * GROUP - k
    if pad:
        wf = torch.nn.functional.pad(wf, (0, pad))
    g = wf.view(n, ng, GROUP)
    scale = (g.abs().amax(dim=2) / 7.0).clamp_min(1e-8).to(torch.float16)
    codes = torch.clamp(torch.round(g / scale.float()[:, :, None]) + 8, 1, 15).to(torch.uint8).view(n, ng * GROUP)[:, :k]
    packed = (codes[:, 0::2] | (codes[:, 1::2] << 4)).contiguous()
    return QuantMatrix(packed, scale.contiguous())


@dataclass
class QuantizedWeights:
    base: DecoderWeights            # embedding, norms, biases, LM head (bf16); its layer matrices are not used
    layers: list                    # per layer: {matrix name: QuantMatrix}

    def to(self, device) -> "QuantizedWeights":
        return QuantizedWeights(self.base.to(device), [{k: m.to(device) for k, m in lw.items()} for lw in self.layers])

    def matrix_bytes(self) -> int:
        return sum(m.nbytes() for lw in self.layers for m in lw.values())


def quantize_weights(w: DecoderWeights) -> QuantizedWeights:
    return QuantizedWeights(w, [{name: quantize_matrix(getattr(lw, name)) for name in MATRICES} for lw in w.layers])
