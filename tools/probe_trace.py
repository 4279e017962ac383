#!/usr/bin/env python
"""Per-task timing of a stream-probe run (no dependencies): body time per op and the gaps between tasks."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.weights import random_weights

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 4
kw = dict(consumer_warps=8, rows_per_tile=64, ktile_chunks=1, n_stage=5)
for a in sys.argv[2:]:
    k, v = a.split("="); kw[k] = int(v)
cfg = PRESETS["qwen2.5-1.5b"]
w = random_weights(cfg, 0, device="cuda")
plug = MegaKernelPlugin(cfg, tt.KernelSchedule(**kw), max_ctx=640)
plug.bind_weights(w)
for _ in range(3):
    plug.stream_probe(mode)
torch.cuda.synchronize()
tr = plug.enable_trace(True)
tr.zero_()
plug.stream_probe(mode)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.float64)
tasks = plug.table.tasks
ran = t[:, 7] > 0
t0 = t[ran][:, 0].min()
print(f"mode {mode}: total {(t[ran][:, 7].max() - t0) / 1e3:.1f} us")
for ty in tuple(tt.GEMV_TYPES) + (tt.T_DOWNK,):
    m = ran & (tasks[:, tt.F_TYPE] == ty)
    if not m.any():
        continue
    d = (t[m][:, 7] - t[m][:, 0]) / 1e3
    byts = np.array([tt.task_weight_bytes(row) for row in tasks[m]], dtype=np.float64) if hasattr(tt, 'task_weight_bytes') else tasks[m][:, tt.F_B].astype(np.float64) * tasks[m][:, tt.F_KCHUNKS] * 512
    print(f"  {tt.TYPE_NAMES[ty]:7s} n={m.sum():6d} body mean {d.mean():7.3f} us  KB/task {byts.mean() / 1e3:8.1f}  -> {byts.sum() / d.sum() / 1e3:7.1f} KB/us per SM")
gaps = []
for sm in range(plug.n_sms):
    lo, hi = plug.table.sm_begin[sm], plug.table.sm_begin[sm + 1]
    idx = [i for i in range(lo, hi) if ran[i]]
    for a, b in zip(idx, idx[1:]):
        gaps.append((t[b, 0] - t[a, 7]) / 1e3)
gaps = np.array(gaps)
print(f"  gaps between consecutive tasks: mean {gaps.mean():.3f} us, p50 {np.median(gaps):.3f}, p95 {np.percentile(gaps, 95):.3f}, total per SM {gaps.sum() / plug.n_sms:.1f} us")
