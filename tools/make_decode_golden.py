#!/usr/bin/env python
"""Generate the decode golden fixtures under tests/golden/ from Hugging Face.

Runs ONLY in the build container (needs ``transformers``; no network: models
are instantiated from a config, weights come from ``weights.random_weights``).
For each tiny preset it loads this repo's random bf16 weights into
``Qwen2ForCausalLM`` / ``Qwen3ForCausalLM`` (fp32 compute, eager attention),
greedy-decodes BASELINE.json configs[0] (16-token prompt, 32 new tokens) and
stores prompt, tokens and per-step logits.  ``tests/test_oracle_decode.py``
pins ``oracle/decode_ref.py`` to these vectors.

    python tools/make_decode_golden.py
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("HF_HUB_OFFLINE", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

from paper_2605_11581_b200.model_config import TINY, TINY_QWEN3, ModelConfig
from paper_2605_11581_b200.weights import DecoderWeights, random_weights


def hf_model(cfg: ModelConfig, w: DecoderWeights):
    import transformers

    common = dict(
        vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.intermediate,
        num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_q_heads,
        num_key_value_heads=cfg.n_kv_heads, rms_norm_eps=cfg.rms_eps, rope_theta=cfg.rope_theta,
        tie_word_embeddings=cfg.tied_embed, max_position_embeddings=4096,
        attn_implementation="eager", use_sliding_window=False,
    )
    if cfg.qk_norm:
        hcfg = transformers.Qwen3Config(head_dim=cfg.head_dim, attention_bias=False, **common)
        model = transformers.Qwen3ForCausalLM(hcfg)
    else:
        hcfg = transformers.Qwen2Config(**common)
        model = transformers.Qwen2ForCausalLM(hcfg)
    sd = {"model.embed_tokens.weight": w.embed, "model.norm.weight": w.final_norm}
    if not cfg.tied_embed:
        sd["lm_head.weight"] = w.lm_head
    for i, l in enumerate(w.layers):
        p = f"model.layers.{i}."
        sd[p + "input_layernorm.weight"] = l.ln1
        sd[p + "post_attention_layernorm.weight"] = l.ln2
        sd[p + "self_attn.q_proj.weight"] = l.wq
        sd[p + "self_attn.k_proj.weight"] = l.wk
        sd[p + "self_attn.v_proj.weight"] = l.wv
        sd[p + "self_attn.o_proj.weight"] = l.wo
        if cfg.qkv_bias:
            sd[p + "self_attn.q_proj.bias"] = l.bq
            sd[p + "self_attn.k_proj.bias"] = l.bk
            sd[p + "self_attn.v_proj.bias"] = l.bv
        if cfg.qk_norm:
            sd[p + "self_attn.q_norm.weight"] = l.q_norm
            sd[p + "self_attn.k_norm.weight"] = l.k_norm
        sd[p + "mlp.gate_proj.weight"] = l.wgate
        sd[p + "mlp.up_proj.weight"] = l.wup
        sd[p + "mlp.down_proj.weight"] = l.wdown
    sd = {k: v.float() for k, v in sd.items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    missing = [m for m in missing if not (cfg.tied_embed and m == "lm_head.weight")]
    assert not missing and not unexpected, (missing, unexpected)
    if cfg.tied_embed:
        model.tie_weights()
    return model.float().eval()


@torch.no_grad()
def hf_greedy(model, prompt: list[int], n_new: int):
    ids = torch.tensor([prompt])
    out = model(ids, use_cache=True)
    past = out.past_key_values
    logits = out.logits[0, -1]
    toks, all_logits = [], []
    for _ in range(n_new):
        all_logits.append(logits.float().numpy().copy())
        nxt = int(torch.argmax(logits))
        toks.append(nxt)
        out = model(torch.tensor([[nxt]]), past_key_values=past, use_cache=True)
        past = out.past_key_values
        logits = out.logits[0, -1]
    return toks, np.stack(all_logits)


def main() -> None:
    out_dir = ROOT / "tests" / "golden"
    out_dir.mkdir(parents=True, exist_ok=True)
    for cfg in (TINY, TINY_QWEN3):
        w = random_weights(cfg, seed=0)
        g = torch.Generator().manual_seed(1)
        prompt = torch.randint(0, cfg.vocab, (16,), generator=g).tolist()
        model = hf_model(cfg, w)
        toks, logits = hf_greedy(model, prompt, 32)
        path = out_dir / f"decode_{cfg.name}.npz"
        np.savez_compressed(path, prompt=np.array(prompt, dtype=np.int32),
                            tokens=np.array(toks, dtype=np.int32),
                            logits=logits[:, :].astype(np.float32))
        srt = np.sort(logits, axis=1)
        print(f"{cfg.name}: tokens {toks[:8]}... distinct {len(set(toks))} "
              f"min top1-top2 margin {float((srt[:, -1] - srt[:, -2]).min()):.4f} -> {path.name}")


if __name__ == "__main__":
    main()
