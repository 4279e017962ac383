#!/usr/bin/env python
"""Per-warp cycle accounting of the stream probes (total / inside gemv_stage / stages)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.weights import random_weights

cfg = PRESETS[sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-1.5b"]
w = random_weights(cfg, 0, device="cuda")
for label, kw in (("c8", dict(consumer_warps=8, rows_per_tile=64, ktile_chunks=1, n_stage=5)),
                  ("c4", dict(consumer_warps=4, rows_per_tile=32, ktile_chunks=2, n_stage=5))):
    plug = MegaKernelPlugin(cfg, tt.KernelSchedule(**kw), max_ctx=640)
    plug.bind_weights(w)
    for mode in (4, 1, 3):
        for _ in range(3):
            plug.stream_probe(mode)
        torch.cuda.synchronize()
        s = plug._sink.view(plug.n_sms, 16, 4)[:, :kw["consumer_warps"]].cpu()
        tot, math, nst, ntask = s[..., 0], s[..., 1], s[..., 2], s[..., 3]
        print(f"{label} probe {mode}: total cyc mean {tot.mean():.0f} max {tot.max():.0f} | math cyc mean {math.mean():.0f} "
              f"({(math / tot).mean():.2f}) | stages/warp {nst.mean():.0f} | cyc/stage {(math / nst).mean():.0f} | tasks {ntask.mean():.0f} "
              f"| non-math per task {((tot - math) / ntask).mean():.0f}")
    plug.close()
