#!/usr/bin/env python
"""Poll anatomy of the gathers (thread 0's first batch): rounds, and when the successful round was issued / returned
relative to the previous phase's last end."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from trace_report import collect
from paper_2605_11581_b200 import task_table as tt

kw = dict(consumer_warps=7, rows_per_tile=42, ktile_chunks=2, n_stage=4, attn_min_chunk=112, l2_prefetch_kb=512, inflight=3)
for a in sys.argv[1:]:
    k, v = a.split("="); kw[k] = int(v)
plug, traces = collect("qwen2.5-1.5b", 512, kw)
tr = traces[-1]
tasks = plug.table.tasks
types, layers = tasks[:, tt.F_TYPE], tasks[:, tt.F_LAYER]
ran = tr[:, 7] > 0
base = float(tr[ran][:, 0].min())
order = [tt.T_QKV, tt.T_ATTN, tt.T_MERGE, tt.T_OPROJ, tt.T_GATEUP, tt.T_DOWN]
acc = {}
prev_end = None
for layer in range(plug.cfg.n_layers):
    for ty in order:
        m = ran & (types == ty) & (layers == layer)
        if not m.any():
            continue
        r = tr[m].astype(np.float64)
        if prev_end is not None and layer >= 1 and ty in (tt.T_QKV, tt.T_OPROJ, tt.T_GATEUP, tt.T_DOWN):
            start = (r[:, 0] - prev_end) / 1e3
            gathered = (r[:, 1] - prev_end) / 1e3
            u = tr[m]
            lo = lambda x: (x & 0xffffffff).astype(np.float64)
            hi = lambda x: (x >> 32).astype(np.float64)
            acc.setdefault(tt.TYPE_NAMES[ty], []).append([np.median(start), np.median(lo(u[:, 3])), np.median(hi(u[:, 3])), np.median(lo(u[:, 4])), np.median(hi(u[:, 4])), np.median(lo(u[:, 6])), np.median(hi(u[:, 6])), np.median(gathered), np.max(gathered)])
        prev_end = tr[m][:, 7].max().astype(np.float64)
print("medians over SMs, mean over layers (us relative to previous phase's last end)")
print(f"{'op':8s} {'start us':>8s} {'stamp':>8s} {'prefetch':>8s} {'erow+flag':>9s} {'load_eop':>8s} {'call':>8s} {'->poll':>8s} (clks) {'gathered us':>12s} {'max':>6s}")
for op, v in acc.items():
    m = np.mean(np.asarray(v), axis=0)
    print(f"{op:8s} " + " ".join(f"{x:8.1f}" for x in m))
