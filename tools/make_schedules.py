#!/usr/bin/env python
"""Offline half -> online half: run the planner's search on the share of a decoder layer one SM executes and
write the SolidifiedTrace the plugin can be built from (paper_2605_11581_b200/schedules/<model>.trace.json).

    python tools/make_schedules.py [model ...]
"""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11581_b200.mkplan import model_graph, search
from paper_2605_11581_b200.model_config import PRESETS

ROOT = Path(__file__).resolve().parents[1] / "paper_2605_11581_b200"
OUT = Path(__file__).resolve().parents[1] / "gpurun_out" / "schedules"   # scratch: a trace placed in
# paper_2605_11581_b200/schedules/<model>.trace.json becomes that model's default schedule (schedules.py)
OUT.mkdir(parents=True, exist_ok=True)
HW = (ROOT / "mkplan" / "fixtures" / "b200.json").read_text()
# B200 search space: tiles of 48-64 rows x 256-512 columns (24-64 KB stages), 2-4 stages, 4-8 consumer warps
SPACE = {"block_m": [16], "block_n": [32, 48, 56, 64], "block_k": [256, 512], "k_split": [1, 2],
         "consumer_warps": [4, 7, 8], "n_stage": [2, 3, 4], "prefetch_stride": [1, 2], "swizzles": [31],
         "flags": {"gap_fill": [False, True]}}

for name in (sys.argv[1:] or ["qwen2.5-1.5b"]):
    cfg = PRESETS[name]
    graph = model_graph.build_sm_slice_graph(cfg, 640)
    t0 = time.time()
    trace = search.run_search(json.dumps(graph), HW, json.dumps(SPACE), 10000)
    text = search.serialize_trace(trace)
    (OUT / f"{name}.trace.json").write_bytes(text if isinstance(text, bytes) else text.encode())
    (OUT / f"{name}.graph.json").write_text(json.dumps(graph, indent=1) + "\n")
    (OUT / "b200.space.json").write_text(json.dumps(SPACE, indent=1) + "\n")
    p = trace.plan
    print(f"{name}: {time.time() - t0:.1f}s  tile {p['tile']} n_stage {p['n_stage']} consumer_warps {p['consumer_warps']} "
          f"stride_eff {p['stride_eff']} duty {trace.score['duty_cycle']:.4f} makespan {trace.score['makespan']} stats {trace.stats}")
