"""GPU check of the batched tensor-core decode (batch_decode.BatchedDecoder) against the CPU oracle + timing.
usage: batch_check.py [quick]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2605_11581_b200.batch_decode import BatchedDecoder
from paper_2605_11581_b200.model_config import PRESETS, TINY, ModelConfig
from paper_2605_11581_b200.weights import random_weights, rope_table

D128_Q3 = ModelConfig(name="test-d128-q3", hidden=512, n_layers=3, n_q_heads=8, n_kv_heads=2, head_dim=128,
                      intermediate=1536, vocab=3000, qkv_bias=False, qk_norm=True, tied_embed=False)


def parity(cfg, B, steps=6, max_ctx=320, oracle_cache=False):
    from oracle.decode_ref import RefDecoder
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, max_ctx)
    ref = RefDecoder(cfg, w, max_ctx, cos, sin, batch=B)
    dec = BatchedDecoder(cfg, w, B, max_ctx)
    g = torch.Generator().manual_seed(11)
    lens = [int(x) for x in torch.randint(3, 280, (B,), generator=g)]
    toks, pos = [], []
    for b in range(B):
        prompt = torch.randint(0, cfg.vocab, (lens[b],), generator=g).tolist()
        ref.prefill(prompt[:-1], b=b) if lens[b] > 1 else None
        dec.prefill(b, prompt)
        toks.append(prompt[-1]); pos.append(lens[b] - 1)
    if oracle_cache:   # isolate the decode step from the (one-ulp different) cache a tensor-core Prefill writes
        dec.k_cache.copy_(ref.k_cache.to(dec.device))
        dec.v_cache.copy_(ref.v_cache.to(dec.device))
    worst = 0.0
    for s in range(steps):
        want = ref.step(toks, pos)
        dec.set_state(toks, pos)
        got_tok = dec.step(auto_advance=False).cpu().tolist()
        got = dec.logits.cpu()
        worst = max(worst, float((got - want).abs().max()))
        toks = [int(t) for t in want.argmax(dim=1)]
        top2 = want.topk(2, dim=1).values
        for b in range(B):
            if float(top2[b, 0] - top2[b, 1]) > 1e-3:
                assert got_tok[b] == toks[b], (s, b, got_tok[b], toks[b])
        pos = [p + 1 for p in pos]
    print(f"{cfg.name} B={B} oracle_cache={oracle_cache}: {steps} steps, max |logit diff| vs oracle {worst:.2e}", flush=True)
    return worst


def bench(name, B, ctx, steps=64, pdl=False, l2_prefetch=False):
    cfg = PRESETS[name]
    w = random_weights(cfg, 0, device="cuda")
    dec = BatchedDecoder(cfg, w, B, ctx + steps * 3 + 16, pdl=pdl, l2_prefetch=l2_prefetch)
    dec.set_state(torch.randint(0, cfg.vocab, (B,)).tolist(), [ctx] * B)
    dec.capture()
    for _ in range(8):
        dec.step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        dec.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    gb = cfg.algorithmic_bytes(ctx, 1) / 1e9
    print(f"{name} batch {B} ctx {ctx} pdl {pdl} l2_prefetch {l2_prefetch}: {ms:.3f} ms/step, {B * 1e3 / ms:.0f} tokens/s, weights once per step -> "
          f"{gb / ms * 1e3:.0f} GB/s of weight streaming ({dec.launches_per_step} own launches/step, CUDA graph)", flush=True)
    del dec


if __name__ == "__main__":
    assert parity(TINY, 3) < 5e-3
    assert parity(D128_Q3, 8) < 5e-3
    assert parity(D128_Q3, 8, oracle_cache=True) < 5e-3
    assert parity(TINY, 5, oracle_cache=True) < 5e-3
    assert parity(D128_Q3, 1) < 5e-3
    if len(sys.argv) > 1 and sys.argv[1] == "quick":
        sys.exit(0)
    bench("qwen2.5-1.5b", 8, 2048, pdl=True)
    bench("qwen2.5-1.5b", 8, 2048, l2_prefetch=True)
    for B in (8, 16, 32, 64, 128):
        bench("qwen2.5-1.5b", B, 2048)
    bench("qwen2.5-7b", 8, 2048)
    bench("qwen2.5-7b", 64, 2048)
