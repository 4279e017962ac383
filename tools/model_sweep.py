#!/usr/bin/env python
"""Decode ms/token of the default schedule, fused vs unfused down projection, for several models.
usage: model_sweep.py [ctx] [model ...]"""
import json
import sys
from dataclasses import replace
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.schedules import default_schedule, fit_schedule
from paper_2605_11581_b200.weights import random_weights

ctx0 = int(sys.argv[1]) if len(sys.argv) > 1 else 512
names = sys.argv[2:] or ["qwen2.5-1.5b", "qwen2.5-7b", "qwen3-8b"]
root = Path(__file__).resolve().parents[1]
peak = json.load(open(root / "MEASURED_PEAKS.json"))["hbm_gbs"] if (root / "MEASURED_PEAKS.json").exists() else 6650.0
steps = 64
for name in names:
    cfg = PRESETS[name]
    w = random_weights(cfg, 0, device="cuda")
    for fuse in (True, False):
        sched = fit_schedule(cfg, replace(default_schedule(cfg), fuse_down=fuse, inflight=0), keep_fused=True)
        plug = MegaKernelPlugin(cfg, sched, max_ctx=ctx0 + steps + 64)
        plug.bind_weights(w)
        kc, vc = plug.kv_view(); kc.normal_(); vc.normal_()
        plug.set_state(1, ctx0)
        for _ in range(5):
            plug.enqueue()
        plug.check()
        plug.set_state(1, ctx0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            plug.enqueue()
        e1.record()
        torch.cuda.synchronize()
        plug.check()
        ms = e0.elapsed_time(e1) / steps
        byts = cfg.algorithmic_bytes(ctx0 + steps // 2)
        print(f"{name:14s} ctx {ctx0} fuse_down {fuse!s:5s} n_stage {sched.n_stage}: {ms * 1e3:8.1f} us/token  {byts / ms / 1e6:7.1f} GB/s = {byts / ms / 1e6 / peak:.3f} of measured HBM peak", flush=True)
        plug.close()
        del plug
    del w
    torch.cuda.empty_cache()
