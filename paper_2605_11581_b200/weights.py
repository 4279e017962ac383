"""Random-init decoder weights in the layout the plugin binds.

There is no network for checkpoints, so every run uses random weights of the
named architecture (BASELINE.json ``configs``).  The init is *scaled*: linear
weights (LM head included) ~ N(0, 1/fan_in), embeddings ~ N(0, 1/hidden) (small
enough that a tied head does not simply echo the input token; logits come out
with std about 1), norm gains 1 + 0.1 N(0, 1), biases ~ N(0, 0.1).  With the plain N(0, 0.02) default a random decoder repeats
one token with tiny logit margins ("Greedy-token identity");
the scaled init keeps every sub-layer's contribution O(1) so the greedy
sequence is non-trivial and argmax margins are far above fp32 reordering noise.

All tensors are bf16 (the storage dtype of the hot path).  Names follow the
Hugging Face Qwen2/Qwen3 module layout so a real checkpoint maps 1:1.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .model_config import ModelConfig


@dataclass
class LayerWeights:
    ln1: torch.Tensor
    wq: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    wo: torch.Tensor
    ln2: torch.Tensor
    wgate: torch.Tensor
    wup: torch.Tensor
    wdown: torch.Tensor
    bq: torch.Tensor | None = None
    bk: torch.Tensor | None = None
    bv: torch.Tensor | None = None
    q_norm: torch.Tensor | None = None
    k_norm: torch.Tensor | None = None

    def tensors(self):
        for name in ("ln1", "wq", "wk", "wv", "bq", "bk", "bv", "q_norm", "k_norm",
                     "wo", "ln2", "wgate", "wup", "wdown"):
            t = getattr(self, name)
            if t is not None:
                yield name, t


@dataclass
class DecoderWeights:
    cfg: ModelConfig
    embed: torch.Tensor
    final_norm: torch.Tensor
    lm_head: torch.Tensor | None  # None when tied to ``embed``
    layers: list[LayerWeights] = field(default_factory=list)

    @property
    def lm_head_matrix(self) -> torch.Tensor:
        return self.embed if self.lm_head is None else self.lm_head

    def to(self, device) -> "DecoderWeights":
        def mv(t):
            return None if t is None else t.to(device)
        layers = [LayerWeights(**{n: mv(getattr(l, n)) for n in LayerWeights.__dataclass_fields__})
                  for l in self.layers]
        return DecoderWeights(self.cfg, mv(self.embed), mv(self.final_norm), mv(self.lm_head), layers)

    def shard(self, rank: int, tp: int) -> "DecoderWeights":
        """The weights of tensor-parallel rank ``rank`` of ``tp`` (``cfg.shard(tp)`` dimensions): q/k/v rows by
        head, O-proj columns by head, gate/up rows and down columns by intermediate channel, LM-head rows by
        vocabulary slice.  ``embed`` stays whole (every rank gathers the input row); norm gains are replicated."""
        if tp == 1:
            return self
        cfg, lc = self.cfg, self.cfg.shard(tp)
        q0, q1 = rank * lc.q_dim, (rank + 1) * lc.q_dim
        k0, k1 = rank * lc.kv_dim, (rank + 1) * lc.kv_dim
        i0, i1 = rank * lc.intermediate, (rank + 1) * lc.intermediate
        v0, v1 = rank * lc.vocab, (rank + 1) * lc.vocab

        def rows(t, a, b):
            return None if t is None else t[a:b].contiguous()

        layers = []
        for l in self.layers:
            layers.append(LayerWeights(
                ln1=l.ln1, wq=rows(l.wq, q0, q1), wk=rows(l.wk, k0, k1), wv=rows(l.wv, k0, k1),
                wo=l.wo[:, q0:q1].contiguous(), ln2=l.ln2, wgate=rows(l.wgate, i0, i1), wup=rows(l.wup, i0, i1),
                wdown=l.wdown[:, i0:i1].contiguous(), bq=rows(l.bq, q0, q1), bk=rows(l.bk, k0, k1), bv=rows(l.bv, k0, k1),
                q_norm=l.q_norm, k_norm=l.k_norm))
        return DecoderWeights(lc, self.embed, self.final_norm, self.lm_head_matrix[v0:v1].contiguous(), layers)

    def n_params(self) -> int:
        n = self.embed.numel() + self.final_norm.numel()
        if self.lm_head is not None:
            n += self.lm_head.numel()
        for l in self.layers:
            n += sum(t.numel() for _, t in l.tensors())
        return n


def random_weights(cfg: ModelConfig, seed: int = 0, device: str | torch.device = "cpu") -> DecoderWeights:
    """Deterministic scaled random init (see module docstring).

    The stream depends on ``device`` type (CPU and CUDA generators differ), so
    parity tests generate once and move the same tensors to both sides.
    """
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)

    def normal(shape, std):
        return (torch.randn(shape, generator=gen, device=dev, dtype=torch.float32) * std).to(torch.bfloat16)

    def gain(n):
        return (1.0 + 0.1 * torch.randn(n, generator=gen, device=dev, dtype=torch.float32)).to(torch.bfloat16)

    h, i, d = cfg.hidden, cfg.intermediate, cfg.head_dim
    embed = normal((cfg.vocab, h), h ** -0.5)
    layers = []
    for _ in range(cfg.n_layers):
        lw = LayerWeights(
            ln1=gain(h),
            wq=normal((cfg.q_dim, h), h ** -0.5),
            wk=normal((cfg.kv_dim, h), h ** -0.5),
            wv=normal((cfg.kv_dim, h), h ** -0.5),
            wo=normal((h, cfg.q_dim), cfg.q_dim ** -0.5),
            ln2=gain(h),
            wgate=normal((i, h), h ** -0.5),
            wup=normal((i, h), h ** -0.5),
            wdown=normal((h, i), i ** -0.5),
        )
        if cfg.qkv_bias:
            lw.bq = normal((cfg.q_dim,), 0.1)
            lw.bk = normal((cfg.kv_dim,), 0.1)
            lw.bv = normal((cfg.kv_dim,), 0.1)
        if cfg.qk_norm:
            lw.q_norm = gain(d)
            lw.k_norm = gain(d)
        layers.append(lw)
    final_norm = gain(h)
    lm_head = None if cfg.tied_embed else normal((cfg.vocab, h), h ** -0.5)
    return DecoderWeights(cfg, embed, final_norm, lm_head, layers)


def rope_table(cfg: ModelConfig, max_ctx: int) -> tuple[torch.Tensor, torch.Tensor]:
    """cos/sin tables [max_ctx, head_dim/2] in fp32.

    Computed exactly as Hugging Face's default rotary embedding does
    (inv_freq = theta^(-2i/d) in fp32, angle = pos * inv_freq in fp32), on the
    CPU, so the device kernel and the CPU oracle consume bit-identical factors.
    """
    half = cfg.head_dim // 2
    inv_freq = 1.0 / (cfg.rope_theta ** (torch.arange(0, cfg.head_dim, 2, dtype=torch.int64).float() / cfg.head_dim))
    pos = torch.arange(max_ctx, dtype=torch.int64).float()
    ang = pos[:, None] * inv_freq[None, :]
    assert ang.shape == (max_ctx, half)
    return ang.cos().contiguous(), ang.sin().contiguous()
