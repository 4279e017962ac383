#!/usr/bin/env python
"""Bring-up benchmark: decode-loop and stream-probe timing for several schedules."""
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
cfg = PRESETS[name]
peak = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))["hbm_gbs"] if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6447.8
t0 = time.time()
w = random_weights(cfg, 0, device="cuda")
torch.cuda.synchronize()
print(f"weights on device in {time.time() - t0:.1f}s", flush=True)
scheds = [
    ("c8 s5 32K pf0", dict(consumer_warps=8, n_stage=5, rows_per_tile=16, ktile_chunks=4, l2_prefetch_kb=0, l2_prefetch_stall_kb=0)),
    ("c8 s5 32K pf128/512", dict(consumer_warps=8, n_stage=5, rows_per_tile=16, ktile_chunks=4)),
    ("c8 s5 32K pf256/1024", dict(consumer_warps=8, n_stage=5, rows_per_tile=16, ktile_chunks=4, l2_prefetch_kb=256, l2_prefetch_stall_kb=1024)),
    ("c8 s5 32K pf64/2048", dict(consumer_warps=8, n_stage=5, rows_per_tile=16, ktile_chunks=4, l2_prefetch_kb=64, l2_prefetch_stall_kb=2048)),
    ("c8 s7 24K", dict(consumer_warps=8, n_stage=7, rows_per_tile=16, ktile_chunks=3)),
    ("c16 s5 32K", dict(consumer_warps=16, n_stage=5, rows_per_tile=32, ktile_chunks=2)),
    ("c16 s3 48K", dict(consumer_warps=16, n_stage=3, rows_per_tile=32, ktile_chunks=3)),
    ("c4 s7 24K", dict(consumer_warps=4, n_stage=7, rows_per_tile=16, ktile_chunks=3)),
]
for label, kw in scheds:
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
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        plug.set_state(1, ctx0)
        e0.record()
        for _ in range(steps):
            plug.enqueue()
        e1.record()
        plug.check()
        ms = e0.elapsed_time(e1) / steps
        for _ in range(3):
            plug.stream_probe()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            plug.stream_probe()
        e1.record()
        torch.cuda.synchronize()
        pms = e0.elapsed_time(e1) / 20
        e0.record()
        for _ in range(20):
            plug.stream_probe(2)
        e1.record()
        torch.cuda.synchronize()
        pms2 = e0.elapsed_time(e1) / 20
        e0.record()
        for _ in range(20):
            plug.stream_probe(3)
        e1.record()
        torch.cuda.synchronize()
        pms3 = e0.elapsed_time(e1) / 20
        byts = cfg.algorithmic_bytes(ctx0 + steps // 2)
        print(f"{label:22s} decode {ms*1e3:8.1f} us/tok {1e3/ms:8.1f} tok/s  {byts/ms/1e6:7.1f} GB/s ({byts/ms/1e6/peak:.3f} of measured)"
              f" | stream probe {pms*1e3:8.1f} us {plug.table.packed_weight_bytes/pms/1e6:7.1f} GB/s"
              f" | loader-only {pms2*1e3:8.1f} us {plug.table.packed_weight_bytes/pms2/1e6:7.1f} GB/s"
              f" | L2-resident {pms3*1e3:8.1f} us {plug.table.packed_weight_bytes/pms3/1e6:7.1f} GB/s", flush=True)
        plug.close()
        del plug
    except Exception as exc:  # keep going: bring-up tool
        print(f"{label}: FAILED {type(exc).__name__}: {exc}", flush=True)
        if "device error" in str(exc) or "CUDA" in str(exc):
            break
