#!/usr/bin/env python
"""Small driver for ncu captures: N decode steps and N stream probes of one schedule."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.weights import random_weights

name, ctx0, mode = sys.argv[1], int(sys.argv[2]), sys.argv[3]
from paper_2605_11581_b200.schedules import default_schedule
kw = None
if len(sys.argv) > 7:
    kw = dict(consumer_warps=int(sys.argv[4]), n_stage=int(sys.argv[5]), rows_per_tile=int(sys.argv[6]),
              ktile_chunks=int(sys.argv[7]))
cfg = PRESETS[name]
w = random_weights(cfg, 0, device="cuda")
plug = MegaKernelPlugin(cfg, tt.KernelSchedule(**kw) if kw else default_schedule(cfg), max_ctx=ctx0 + 64)
plug.bind_weights(w)
kc, vc = plug.kv_view(); kc.normal_(); vc.normal_()
plug.set_state(1, ctx0)
for _ in range(12):
    if mode == "decode":
        plug.enqueue()
    else:
        plug.stream_probe(int(mode))
plug.check()
print("done")
