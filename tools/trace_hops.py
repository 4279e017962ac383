#!/usr/bin/env python
"""Distribution over SMs of 'inputs gathered' and 'task end' times relative to the previous phase's last end."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from trace_report import collect
from paper_2605_11581_b200 import task_table as tt

kw = dict(consumer_warps=7, rows_per_tile=42, ktile_chunks=2, n_stage=4, attn_min_chunk=112, l2_prefetch_kb=512)
for a in sys.argv[1:]:
    k, v = a.split("="); kw[k] = int(v)
plug, traces = collect("qwen2.5-1.5b", 512, kw)
tr = traces[-1]
tasks = plug.table.tasks
types, layers = tasks[:, tt.F_TYPE], tasks[:, tt.F_LAYER]
ran = tr[:, 7] > 0
rel = (tr.astype(np.float64) - float(tr[ran][:, 0].min())) / 1e3
order = [tt.T_QKV, tt.T_ATTN, tt.T_MERGE, tt.T_OPROJ, tt.T_GATEUP, tt.T_DOWN]
pct = (0, 25, 50, 75, 90, 99, 100)
acc = {}
prev_end = None
for layer in range(plug.cfg.n_layers):
    for ty in order:
        m = ran & (types == ty) & (layers == layer)
        if not m.any():
            continue
        r = rel[m]
        if prev_end is not None and layer >= 1:
            g = (r[:, 1] if ty != tt.T_MERGE else r[:, 0]) - prev_end
            e = r[:, 7] - prev_end
            acc.setdefault(tt.TYPE_NAMES[ty], []).append((np.percentile(g, pct), np.percentile(e, pct)))
        prev_end = r[:, 7].max()
print("percentiles over SMs", pct, "(us after the previous phase's last end; mean over layers)")
for op, v in acc.items():
    g = np.mean([x[0] for x in v], axis=0); e = np.mean([x[1] for x in v], axis=0)
    print(f"{op:7s} gathered " + " ".join(f"{x:6.2f}" for x in g) + "   | end " + " ".join(f"{x:6.2f}" for x in e))
