"""Oracle half of the W4A16 path: the reference dequantisation.  TEST INFRASTRUCTURE -- only tests/, smoke() and
bench.py's CPU leg may import this; the product path (paper_2605_11581_b200/) never does.

The reference states the format as a byte model only (``/root/reference/pkg/src/mkplan/graph_ir.py:296-318``: 4-bit
codes, ``INT4_GROUP_SIZE = 128``, two bytes per scale); the arithmetic is GPTQ's published dequantisation with a
fixed zero point of 8:  ``W[n][k] = (code[n][k] - 8) * scale[n][k // 128]``, evaluated in fp32 (a 4-bit integer times
an fp16 value is exact in fp32).  Parity is pinned by the identity ``dequant(quantize(W))`` round trip and by the byte
model (``tests/test_w4a16.py``); the decode arithmetic around it is the oracle of ``decode_ref.py``."""

from __future__ import annotations

import copy

import torch

GROUP = 128


def dequant_w4a16(q: torch.Tensor, s: torch.Tensor) -> torch.Tensor:
    """codes uint8 [N, K / 2] (even k in the low nibble), scales fp16 [N, ceil(K / 128)] -> fp32 [N, K]."""
    q = q.cpu()
    n, half = q.shape
    codes = torch.empty(n, half * 2, dtype=torch.float32)
    codes[:, 0::2] = (q & 15).float()
    codes[:, 1::2] = (q >> 4).float()
    scale = s.cpu().float().repeat_interleave(GROUP, dim=1)[:, :half * 2]
    return (codes - 8.0) * scale


def dequantized_weights(qw):
    """A DecoderWeights whose layer matrices are the fp32 dequantisation of ``qw`` (what RefDecoder multiplies)."""
    w = copy.copy(qw.base)
    w.layers = []
    for lw, ql in zip(qw.base.layers, qw.layers):
        new = copy.copy(lw)
        for name, m in ql.items():
            setattr(new, name, dequant_w4a16(m.q, m.s))
        w.layers.append(new)
    return w
