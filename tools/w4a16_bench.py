#!/usr/bin/env python
"""W4A16 decode: ms/token and the fraction of the int4 weight-streaming roofline (codes + scales + bf16 LM head + KV).

    python tools/w4a16_bench.py [model] [ctx] [steps]
"""
import json
import sys
from dataclasses import replace
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import quant
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.schedules import default_schedule, fit_schedule
from paper_2605_11581_b200.weights import random_weights

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-1.5b"
ctx0 = int(sys.argv[2]) if len(sys.argv) > 2 else 512
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 128
cfg = PRESETS[name]
root = Path(__file__).resolve().parents[1]
peak = json.load(open(root / "MEASURED_PEAKS.json"))["hbm_gbs"] if (root / "MEASURED_PEAKS.json").exists() else 6650.0
w = random_weights(cfg, 0)
qw = quant.quantize_weights(w)


def timed(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for label, weights, w4 in (("bf16", w, False), ("w4a16", qw, True)):
    sched = fit_schedule(cfg, replace(default_schedule(cfg), fuse_down=True, w4a16=w4, inflight=0), keep_fused=True)
    plug = MegaKernelPlugin(cfg, sched, max_ctx=ctx0 + steps + 64)
    plug.bind_weights(weights)
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
    kv = cfg.algorithmic_bytes(ctx0 + steps // 2) - cfg.weight_bytes_per_token()
    if w4:
        lm = cfg.vocab * cfg.hidden * 2
        norms = cfg.weight_bytes_per_token() - lm * (1 if True else 0) - sum(getattr(lw, n).numel() * 2 for lw in w.layers for n in quant.MATRICES)
        algo = qw.matrix_bytes() + lm + max(norms, 0) + kv
    else:
        algo = cfg.algorithmic_bytes(ctx0 + steps // 2)
    print(f"{label:6s} {name} ctx {ctx0}: {ms * 1e3:7.1f} us/token {1e3 / ms:7.1f} tok/s | algorithmic bytes {algo / 1e9:.3f} GB -> {algo / ms / 1e6:7.1f} GB/s "
          f"= {algo / ms / 1e6 / peak:.3f} of the measured HBM peak | packed stream {plug.table.packed_weight_bytes / 1e9:.3f} GB | "
          f"stream probe {pr * 1e3:.1f} us ({plug.table.packed_weight_bytes / pr / 1e6:.0f} GB/s)", flush=True)
    plug.close()
    del plug
