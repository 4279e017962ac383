"""SPEC.md:509 at full model dimensions: `mkplan search` over ONE WHOLE Qwen2.5-1.5B decoder layer (hidden 1536,
intermediate 8960, 12/2 heads, context 512 -- 384 908 micro-ops and 1.1 M RAW edges at tile 16x128x128, k_split 2;
the reference planner needs ~25-30 min per candidate on such a graph) with worker processes
(MK_PLANNER_PROCS).  Prints the wall-clock time, the stats and the content hash; run twice with different process
counts the hash must not change.
usage: full_dim_search.py [procs] [out.trace]"""
import json
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11581_b200.mkplan import model_graph, search
from paper_2605_11581_b200.model_config import get_config

SPACE = {"block_m": [16], "block_n": [128], "block_k": [128], "k_split": [1, 2], "consumer_warps": [4, 8],
         "n_stage": [2, 3, 4], "prefetch_stride": [1, 2], "swizzles": [3], "flags": {"gap_fill": [False, True]}}

if __name__ == "__main__":
    procs = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
    os.environ["MK_PLANNER_PROCS"] = str(procs)
    graph = model_graph.layer_graph_json(get_config("qwen2.5-1.5b"), 512)
    hw = (Path(search.__file__).parent / "fixtures" / "b200.json").read_text()
    t0 = time.time()
    trace = search.run_search(graph, hw, json.dumps(SPACE), 10000)
    dt = time.time() - t0
    ops = len(trace.candidate.trace.ops)
    print(f"full-dimension layer search: {dt:.1f} s with {procs} worker processes; winner tile {trace.plan['tile']} "
          f"({ops} micro-ops), n_stage {trace.plan['n_stage']}, warps {trace.plan['consumer_warps']}, stats {trace.stats}, "
          f"duty {trace.score['duty_cycle']:.4f}, makespan {trace.score['makespan']}, content_hash {trace.content_hash}")
    if len(sys.argv) > 2:
        Path(sys.argv[2]).write_bytes(search.serialize_trace(trace))
