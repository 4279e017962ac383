#!/usr/bin/env python
"""GPU bring-up helper: run a few decode steps and print per-buffer diffs vs the oracle."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from oracle.decode_ref import RefDecoder
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import PRESETS, ModelConfig
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.weights import random_weights, rope_table

name = sys.argv[1] if len(sys.argv) > 1 else "tiny-qwen2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
cfg = PRESETS[name]
sched = tt.KernelSchedule(consumer_warps=8, n_stage=4, rows_per_tile=16, ktile_chunks=2, attn_min_chunk=8)
w = random_weights(cfg, 0)
cos, sin = rope_table(cfg, 128)
ref = RefDecoder(cfg, w, 128, cos, sin)
plug = MegaKernelPlugin(cfg, sched, max_ctx=128)
print("table", plug.table.summary())
plug.bind_weights(w)
want_p = tt.pack_weights_reference(plug.table, w)
got_p = plug.packed[:plug.table.packed_weight_bytes].cpu().numpy().view(np.uint16)
print("packer mismatches:", int((want_p != got_p).sum()), "of", want_p.size)
g = torch.Generator().manual_seed(1)
toks = torch.randint(0, cfg.vocab, (steps,), generator=g).tolist()
for pos, tok in enumerate(toks):
    want = ref.step([tok], [pos])[0].numpy()
    out = plug.decode_step(tok, pos)
    plug.check()
    got = out.logits[0].cpu().numpy()
    print(f"pos {pos}: max|d|={np.abs(got - want).max():.3e} argmax {int(out.next_token.item())} vs {int(want.argmax())}"
          f" nan={int(np.isnan(got).sum())}")
print("OK")
