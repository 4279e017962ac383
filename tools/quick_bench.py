#!/usr/bin/env python
"""Bring-up benchmark: decode-loop and stream-probe timing for several schedules.

usage: quick_bench.py [model] [ctx] [steps] [filter]
"""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.weights import random_weights

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-1.5b"
ctx0 = int(sys.argv[2]) if len(sys.argv) > 2 else 512
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 64
flt = sys.argv[4] if len(sys.argv) > 4 else ""
cfg = PRESETS[name]
root = Path(__file__).resolve().parents[1]
peak = json.load(open(root / "MEASURED_PEAKS.json"))["hbm_gbs"] if (root / "MEASURED_PEAKS.json").exists() else 6650.0
t0 = time.time()
w = random_weights(cfg, 0, device="cuda")
torch.cuda.synchronize()
print(f"weights on device in {time.time() - t0:.1f}s", flush=True)
B = dict(consumer_warps=8, rows_per_tile=64, ktile_chunks=1, n_stage=5, attn_min_chunk=64)
C4 = dict(B, consumer_warps=4, rows_per_tile=32)
C7 = dict(B, consumer_warps=7, attn_min_chunk=128)
D7 = dict(C7, rows_per_tile=56, ktile_chunks=2, n_stage=3, l2_prefetch_kb=512)
D7 = dict(C7, l2_prefetch_kb=512, attn_min_chunk=112)
D7 = dict(C7, l2_prefetch_kb=512, attn_min_chunk=112, rows_per_tile=42, ktile_chunks=2, n_stage=4)
D7 = dict(consumer_warps=7, rows_per_tile=42, ktile_chunks=2, n_stage=5, attn_min_chunk=112, l2_prefetch_kb=512)
scheds = [
    ("fused", dict(D7, inflight=3, fuse_down=True)),
    ("base", dict(D7)),
    ("if3", dict(D7, inflight=3)),
    ("if2", dict(D7, inflight=2)),
    ("pf1024", dict(D7, l2_prefetch_kb=1024)),
    ("if3 pf1024", dict(D7, inflight=3, l2_prefetch_kb=1024)),
    ("if3 pf1024 mc168", dict(D7, inflight=3, l2_prefetch_kb=1024, attn_min_chunk=168)),
    ("if3 pf2048", dict(D7, inflight=3, l2_prefetch_kb=2048)),
]


def timed(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for label, kw in scheds:
    if flt and flt not in label:
        continue
    try:
        sched = tt.KernelSchedule(**kw)
        plug = MegaKernelPlugin(cfg, sched, max_ctx=ctx0 + steps + 64)
        plug.bind_weights(w)
        kc, vc = plug.kv_view()
        kc.normal_(); vc.normal_()
        plug.set_state(1, ctx0)
        for _ in range(5):
            plug.enqueue()
        plug.check()
        plug.set_state(1, ctx0)
        ms = timed(plug.enqueue, steps)
        plug.check()
        probes = {}
        for mode, nm in ((1, "stream"), (2, "loader-only"), (3, "L2-resident"), (4, "consumer-only")):
            for _ in range(3):
                plug.stream_probe(mode)
            torch.cuda.synchronize()
            probes[nm] = timed(lambda: plug.stream_probe(mode), 20)
        byts = cfg.algorithmic_bytes(ctx0 + steps // 2)
        pw = plug.table.packed_weight_bytes
        print(f"{label:18s} decode {ms*1e3:8.1f} us/tok {1e3/ms:8.1f} tok/s  {byts/ms/1e6:7.1f} GB/s ({byts/ms/1e6/peak:.3f} of measured) | "
              + " | ".join(f"{nm} {v*1e3:7.1f} us {pw/v/1e6:7.1f} GB/s" for nm, v in probes.items()), flush=True)
        plug.close()
        del plug
    except Exception as exc:  # keep going: bring-up tool
        print(f"{label}: FAILED {type(exc).__name__}: {exc}", flush=True)
        if "device error" in str(exc) or "CUDA" in str(exc):
            break
