#!/usr/bin/env python
"""Batch sweep on the CUDA-core path (plugin.BatchLanes): tokens/s of `batch` sequences decoded concurrently on
disjoint SM partitions that stream one packed weight buffer.  usage: batch_sweep.py [model] [ctx] [steps]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import BatchLanes
from paper_2605_11581_b200.schedules import default_schedule
from paper_2605_11581_b200.weights import random_weights

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-1.5b"
ctx0 = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 32
cfg = PRESETS[name]
w = random_weights(cfg, 0, device="cuda")
for batch in (1, 2, 4, 8):
    lanes = BatchLanes(cfg, default_schedule(cfg), max_ctx=ctx0 + steps + 16, batch=batch)
    lanes.bind_weights(w)
    for lane in lanes.lanes:
        kc, vc = lane.kv_view(); kc.normal_(); vc.normal_()
    lanes.set_state([1] * batch, [ctx0] * batch)
    for _ in range(4):
        lanes.enqueue()
    lanes.check()
    lanes.set_state([1] * batch, [ctx0] * batch)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        lanes.enqueue()
    e1.record()
    lanes.check()
    ms = e0.elapsed_time(e1) / steps
    byts = cfg.weight_bytes_per_token() + batch * (ctx0 + steps // 2) * cfg.kv_bytes_per_ctx_token()
    print(f"{name} ctx {ctx0} batch {batch}: {ms * 1e3:8.1f} us/step  {batch * 1e3 / ms:8.1f} tok/s  "
          f"{byts / ms / 1e6:7.1f} GB/s algorithmic ({lanes.lanes[0].n_sms} SMs per lane)", flush=True)
    lanes.close()
