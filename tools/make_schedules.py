#!/usr/bin/env python
"""Offline half -> online half: run the planner's search on the share of a decoder layer one SM executes and
write the SolidifiedTrace the kernel is built from (paper_2605_11581_b200/schedules/<model>.{trace,graph,space,hw,kernel}.json).

Two steps, as the paper solidifies its path (the search proposes, offline profiling on the target
GPU locks the trace in):

  1. ``--survey``: the WIDE B200 space (every tile the kernel can run with seven or eight consumer warps) is searched
     and the best candidate per tile is listed with its simulated score -- these are the candidates to profile
     (``tools/pace_sweep.py`` / ``profiles/r02_schedule_candidates.md`` hold the measurements).
  2. default: the NARROW space around the profiled tile is searched; the winner -- pipeline depth, prefetch stride,
     passes -- is the shipped trace.  The reference planner produces the same bytes from the same three files
     (tests/test_schedules.py).

    python tools/make_schedules.py [--survey] [model ...]
"""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11581_b200.mkplan import model_graph, search
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.solidify import check_program_order

ROOT = Path(__file__).resolve().parents[1] / "paper_2605_11581_b200"
OUT = ROOT / "schedules"
HW = (ROOT / "mkplan" / "fixtures" / "b200.json").read_text()
CTX = 640          # the bench's context (512-token prompt + 128 decode steps)
BUDGET = 10000
# every tile the kernel runs with 7 (8 warps per CTA: full register budget) or 8 consumer warps
WIDE = {"block_m": [16], "block_n": [32, 48, 56, 64], "block_k": [256, 512], "k_split": [1, 2],
        "consumer_warps": [7, 8], "n_stage": [2, 3, 4, 5], "prefetch_stride": [1, 2, 3], "swizzles": [31],
        "flags": {"gap_fill": [False, True]}}
# the profiled tile (profiles/r02_schedule_candidates.md): 48 x 512 on seven warps = 42-row kernel tiles
NARROW = {"block_m": [16], "block_n": [48], "block_k": [512], "k_split": [1], "consumer_warps": [7],
          "n_stage": [2, 3, 4], "prefetch_stride": [1, 2], "swizzles": [31], "flags": {"gap_fill": [False, True]}}
# run-time knobs the planner does not model
KERNEL = {"attn_min_chunk": 112, "l2_prefetch_kb": 512, "fuse_down": True, "poll_inflight": 9}
# the fused K-slice down projection pays only with one 256-row block per consumer warp (tools/model_sweep.py)
# (and holding ring fills while the consumers poll measures 0.6 % slower on them, 1.2 % faster on the 1.5B)
BIG = {"attn_min_chunk": 112, "l2_prefetch_kb": 512, "fuse_down": False}
KERNEL_BY_MODEL = {"qwen2.5-7b": BIG, "qwen3-8b": BIG}


def main() -> None:
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    survey = "--survey" in sys.argv
    OUT.mkdir(parents=True, exist_ok=True)
    for name in (args or ["qwen2.5-1.5b"]):
        cfg = PRESETS[name]
        graph_text = json.dumps(model_graph.build_sm_slice_graph(cfg, CTX, page_bytes=json.loads(HW)["page_size_bytes"]), indent=1) + "\n"
        if survey:
            t0 = time.time()
            trace = search.run_search(graph_text, HW, json.dumps(WIDE), BUDGET, debug=True)
            best: dict = {}
            for e in trace.entries:
                key = tuple(e.candidate.tile.key()) + (e.candidate.consumer_warps,)
                if key not in best or e.order_key() < best[key].order_key():
                    best[key] = e
            print(f"{name}: wide space, {trace.stats} in {time.time() - t0:.1f}s; best candidate per (tile, warps):")
            for key, e in sorted(best.items(), key=lambda kv: kv[1].order_key()):
                print(f"  tile {list(key[:4])} warps {key[4]} n_stage {e.candidate.n_stage} stride {e.candidate.prefetch_stride} "
                      f"duty {e.duty:.4f} makespan {e.makespan}")
            continue
        t0 = time.time()
        space_text = json.dumps(NARROW, indent=1) + "\n"
        trace = search.run_search(graph_text, HW, space_text, BUDGET)
        text = search.serialize_trace(trace)
        text = text if isinstance(text, bytes) else text.encode()
        (OUT / f"{name}.trace.json").write_bytes(text)
        (OUT / f"{name}.graph.json").write_text(graph_text)
        (OUT / f"{name}.space.json").write_text(space_text)
        (OUT / f"{name}.hw.json").write_text(HW)
        (OUT / f"{name}.kernel.json").write_text(json.dumps(KERNEL_BY_MODEL.get(name, KERNEL), indent=1) + "\n")
        order = check_program_order(search.parse_trace(text), graph_text, HW)
        p = trace.plan
        print(f"{name}: {time.time() - t0:.1f}s  tile {p['tile']} n_stage {p['n_stage']} consumer_warps {p['consumer_warps']} "
              f"stride_eff {p['stride_eff']} per_stage {p['per_stage']} window {p['window']} duty {trace.score['duty_cycle']:.4f} "
              f"makespan {trace.score['makespan']} stats {trace.stats} content_hash {trace.content_hash[:16]} order {order}")


if __name__ == "__main__":
    main()
