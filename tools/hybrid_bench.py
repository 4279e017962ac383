#!/usr/bin/env python
"""BASELINE.json configs[4]: hybrid engine end-to-end latency -- Qwen2.5-7B, 4K-token prompt, 256 generated
tokens; prefill on the hand-written tensor-core backend (prefill.py; 1 or 2 activation planes) or on the library
backend (bf16 cuBLAS GEMMs + library attention, the baseline), decode on the MegaKernel.
usage: hybrid_bench.py [model] [prompt] [new_tokens] [tensor1|tensor2|library]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200.engine import HybridEngine
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.weights import random_weights

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
n_prompt = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
n_new = int(sys.argv[3]) if len(sys.argv) > 3 else 256
mode = sys.argv[4] if len(sys.argv) > 4 else "tensor1"
cfg = PRESETS[name]
w = random_weights(cfg, 0, device="cuda")
if mode == "library":
    eng = HybridEngine(cfg, w, max_ctx=n_prompt + n_new + 16, prefill_backend="library", prefill_dtype=torch.bfloat16)
else:
    eng = HybridEngine(cfg, w, max_ctx=n_prompt + n_new + 16, prefill_backend="tensor", prefill_planes=int(mode[-1]), prefill_attention="bf16")
g = torch.Generator().manual_seed(1)
prompt = torch.randint(0, cfg.vocab, (n_prompt,), generator=g).tolist()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.prefill(prompt)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if rep == 1:
        continue
    res = eng.generate(prompt, n_new) if rep == 0 else None
    if rep == 2:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n_new):
            eng.plugin.enqueue()
        e1.record()
        eng.plugin.check()
        dec_ms = e0.elapsed_time(e1)
        print(f"{name}: prefill {n_prompt} tokens ({mode}) {1e3 * (t1 - t0):.1f} ms | decode {n_new} tokens "
              f"{dec_ms:.1f} ms ({dec_ms / n_new:.3f} ms/token) | end to end {1e3 * (t1 - t0) + dec_ms:.1f} ms")
eng.close()
