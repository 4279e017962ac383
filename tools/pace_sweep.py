#!/usr/bin/env python
"""Loader pacing sweep: decode time per token against the aggregate HBM request rate the Loaders are metered to.

usage: pace_sweep.py [model] [ctx] [steps] [key=value ...]   (extra KernelSchedule fields)
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.weights import random_weights

pos_args = [a for a in sys.argv[1:] if "=" not in a]
name = pos_args[0] if len(pos_args) > 0 else "qwen2.5-1.5b"
ctx0 = int(pos_args[1]) if len(pos_args) > 1 else 512
steps = int(pos_args[2]) if len(pos_args) > 2 else 128
extra = {}
rates = [0, 5000, 5500, 6000, 6500, 7000, 7500]
for a in sys.argv[1:]:
    if "=" in a:
        k, v = a.split("=")
        if k == "rates":
            rates = [int(x) for x in v.split(",")]
        else:
            extra[k] = int(v)
cfg = PRESETS[name]
w = random_weights(cfg, 0, device="cuda")
base = dict(consumer_warps=7, rows_per_tile=42, ktile_chunks=2, n_stage=4, attn_min_chunk=112, l2_prefetch_kb=512, inflight=3)
base.update(extra)


def timed(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for gbs in rates:
    kw = dict(base, pace_clk_per_64k=tt.pace_for(gbs))
    plug = MegaKernelPlugin(cfg, tt.KernelSchedule(**kw), max_ctx=ctx0 + steps + 64)
    plug.bind_weights(w)
    kc, vc = plug.kv_view(); kc.normal_(); vc.normal_()
    plug.set_state(1, ctx0)
    for _ in range(5):
        plug.enqueue()
    plug.check()
    plug.set_state(1, ctx0)
    ms = timed(plug.enqueue, steps)
    plug.check()
    for _ in range(3):
        plug.stream_probe(1)
    torch.cuda.synchronize()
    pr = timed(lambda: plug.stream_probe(1), 20)
    print(f"pace {gbs:5d} GB/s (clk/64K {kw['pace_clk_per_64k']:5d}) {extra}: decode {ms*1e3:7.1f} us/tok | stream probe {pr*1e3:7.1f} us", flush=True)
    plug.close()
    del plug
