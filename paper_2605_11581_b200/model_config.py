"""Decoder model configurations for the decode MegaKernel path.

The reference ships no model description: its only statement of what a decode
step contains is the operator-kind list (reference
``pkg/src/mkplan/graph_ir.py:48-56``) and the paper's layer walk
(``PAPER.md:216-218``).  ``ModelConfig`` carries the Qwen2 / Qwen2.5 / Qwen3
dimensions named by BASELINE.json and SURVEY.md section 8(d); everything
downstream (operator-graph builder, device task table, plugin) is derived from
it.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass


@dataclass(frozen=True)
class ModelConfig:
    name: str
    hidden: int
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int
    rms_eps: float = 1e-6
    rope_theta: float = 1e6
    qkv_bias: bool = True      # Qwen2 / Qwen2.5
    qk_norm: bool = False      # Qwen3
    tied_embed: bool = True

    def __post_init__(self) -> None:
        if self.n_q_heads % self.n_kv_heads:
            raise ValueError("n_q_heads must be a multiple of n_kv_heads")
        if self.head_dim not in (64, 128):
            raise ValueError("head_dim must be 64 or 128")
        for f in ("hidden", "n_layers", "n_q_heads", "n_kv_heads", "intermediate", "vocab"):
            if getattr(self, f) <= 0:
                raise ValueError(f"{f} must be positive")

    @property
    def q_dim(self) -> int:
        return self.n_q_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    @property
    def group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    @property
    def qkv_rows(self) -> int:
        return self.q_dim + 2 * self.kv_dim

    def layer_weight_elems(self) -> int:
        """bf16 matrix + vector elements one layer streams per decoded token."""
        h, i = self.hidden, self.intermediate
        n = self.qkv_rows * h + h * self.q_dim + 2 * i * h + h * i + 2 * h
        if self.qkv_bias:
            n += self.qkv_rows
        if self.qk_norm:
            n += 2 * self.head_dim
        return n

    def weight_bytes_per_token(self) -> int:
        """Algorithmic weight bytes per decoded token: every
        layer weight, the final norm and the LM head read once, bf16."""
        elems = self.n_layers * self.layer_weight_elems() + self.hidden + self.vocab * self.hidden
        return 2 * elems

    def kv_bytes_per_ctx_token(self) -> int:
        return 2 * self.kv_dim * 2 * self.n_layers

    def algorithmic_bytes(self, ctx: int, batch: int = 1) -> int:
        return self.weight_bytes_per_token() + batch * ctx * self.kv_bytes_per_ctx_token()

    def shard(self, tp: int) -> "ModelConfig":
        """Dimensions of ONE tensor-parallel rank (Megatron-style): q/k/v heads, the MLP
        intermediate channels and the LM-head vocabulary are split ``tp`` ways; ``hidden`` is not."""
        if tp == 1:
            return self
        if tp not in (2, 4, 8):
            raise ValueError("tp must be 1, 2, 4 or 8")
        for f in ("n_q_heads", "n_kv_heads", "intermediate", "vocab"):
            if getattr(self, f) % tp:
                raise ValueError(f"{f}={getattr(self, f)} is not divisible by tp={tp}")
        if (self.intermediate // tp) % 8:
            raise ValueError("intermediate / tp must be a multiple of 8")
        from dataclasses import replace
        return replace(self, name=f"{self.name}-tp{tp}", n_q_heads=self.n_q_heads // tp, n_kv_heads=self.n_kv_heads // tp,
                       intermediate=self.intermediate // tp, vocab=self.vocab // tp)

    def to_dict(self) -> dict:
        return asdict(self)


# BASELINE.json configs[0]: runs on the CPU oracle.  intermediate=704 is this
# repo's documented choice; it is not a multiple of 256, which
# exercises the K-padding path of the weight packer.
TINY = ModelConfig(
    name="tiny-qwen2", hidden=256, n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=64,
    intermediate=704, vocab=1024,
)
# Same shape family with QK-norm and no bias / untied head (Qwen3 flavour).
TINY_QWEN3 = ModelConfig(
    name="tiny-qwen3", hidden=256, n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=64,
    intermediate=704, vocab=1024, qkv_bias=False, qk_norm=True, tied_embed=False,
)
QWEN25_1P5B = ModelConfig(
    name="qwen2.5-1.5b", hidden=1536, n_layers=28, n_q_heads=12, n_kv_heads=2, head_dim=128,
    intermediate=8960, vocab=151936,
)
QWEN25_7B = ModelConfig(
    name="qwen2.5-7b", hidden=3584, n_layers=28, n_q_heads=28, n_kv_heads=4, head_dim=128,
    intermediate=18944, vocab=152064, tied_embed=False,
)
QWEN3_8B = ModelConfig(
    name="qwen3-8b", hidden=4096, n_layers=36, n_q_heads=32, n_kv_heads=8, head_dim=128,
    intermediate=12288, vocab=151936, qkv_bias=False, qk_norm=True, tied_embed=False,
)

PRESETS = {c.name: c for c in (TINY, TINY_QWEN3, QWEN25_1P5B, QWEN25_7B, QWEN3_8B)}


def get_config(name: str) -> ModelConfig:
    try:
        return PRESETS[name]
    except KeyError as exc:
        raise KeyError(f"unknown model preset {name!r}; have {sorted(PRESETS)}") from exc
