import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from dataclasses import replace
from oracle.decode_ref import RefDecoder
from paper_2605_11581_b200.model_config import QWEN3_8B, QWEN25_7B
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.schedules import default_schedule, fit_schedule
from paper_2605_11581_b200.weights import random_weights, rope_table
variants = [replace(QWEN3_8B, n_layers=1, name="q3"), replace(QWEN3_8B, n_layers=1, qk_norm=False, name="q3-nonorm"),
            replace(QWEN25_7B, n_layers=1, qk_norm=True, qkv_bias=False, name="q25-norm"),
            replace(QWEN3_8B, n_layers=1, vocab=4096, name="q3-smallvocab"),
            replace(QWEN3_8B, n_layers=1, intermediate=8192, name="q3-I8192"),
            replace(QWEN3_8B, n_layers=1, n_q_heads=16, n_kv_heads=4, name="q3-16h")]
for cfg in variants:
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, 32)
    ref = RefDecoder(cfg, w, 32, cos, sin)
    toks = [5, 77]
    wants = [ref.step([t], [p])[0].numpy() for p, t in enumerate(toks)]
    sched = default_schedule(cfg)
    plug = MegaKernelPlugin(cfg, sched, max_ctx=32)
    plug.bind_weights(w)
    errs = []
    for p, t in enumerate(toks):
        out = plug.decode_step(t, p, want_logits=True); plug.check()
        errs.append(float(np.abs(out.logits[0].cpu().numpy() - wants[p]).max()))
    kc, vc = plug.kv_view()
    dk = float((kc[:, 0, :, :2].float().cpu() - ref.k_cache[:, 0, :, :2].float()).abs().max())
    dv = float((vc[:, 0, :, :2].float().cpu() - ref.v_cache[:, 0, :, :2].float()).abs().max())
    print(cfg.name, "errs", ["%.2e" % e for e in errs], "kv diff %.2e %.2e" % (dk, dv), flush=True)
    plug.close(); del plug
