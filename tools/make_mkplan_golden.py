#!/usr/bin/env python
"""Generate planner golden files by RUNNING THE REFERENCE (build container only).

Imports the unmodified reference package from /root/reference/pkg/src (module
name ``mkplan``) and records, for a fixed set of graph / hardware / search-space
inputs, the exact bytes it produces: solidified traces, DOT graphs, ``lower``
summaries, simulation reports, CLI text and exit codes.  The inputs themselves
are written next to the outputs, so tests/test_mkplan_parity.py needs nothing
but tests/golden/mkplan/ (the GPU box has no /root/reference).

    python tools/make_mkplan_golden.py [--quick]
"""

from __future__ import annotations

import contextlib
import io
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(REF))

import mkplan  # the reference  # noqa: E402
from mkplan import cli as ref_cli  # noqa: E402

from paper_2605_11581_b200.mkplan.model_graph import build_layer_graph  # noqa: E402
from paper_2605_11581_b200.model_config import TINY, ModelConfig  # noqa: E402

assert Path(mkplan.__file__).is_relative_to(REF), mkplan.__file__
OUT = ROOT / "tests" / "golden" / "mkplan"
FIX = ROOT / "paper_2605_11581_b200" / "mkplan" / "fixtures"

PROBE = ModelConfig(name="probe-256", hidden=256, n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=64,
                    intermediate=512, vocab=1024)
FLAGS_ALL = {k: [False, True] for k in ("gap_fill", "reuse_act_weight", "reuse_act_output", "split_reduction")}

SPACES = {
    # the 2 304-point tiny-gemm space
    "tiny-full": {"block_m": [16], "block_n": [8], "block_k": [16], "k_split": [1, 2], "consumer_warps": [4, 8, 16],
                  "n_stage": [1, 2, 3, 4], "prefetch_stride": [1, 2, 3], "swizzles": [0, 31], "flags": FLAGS_ALL},
    # SURVEY.md appendix A
    "layer-a": {"block_m": [16], "block_n": [64], "block_k": [64], "k_split": [1, 2], "consumer_warps": [8, 16],
                "n_stage": [2, 4], "prefetch_stride": [1, 2], "swizzles": [0, 31],
                "flags": {"gap_fill": [False, True], "reuse_act_weight": [False, True], "reuse_act_output": [False],
                          "split_reduction": [False, True]}},
    "layer-small": {"block_m": [16], "block_n": [64], "block_k": [128], "k_split": [1, 2], "consumer_warps": [8],
                    "n_stage": [2, 3], "prefetch_stride": [1, 2], "swizzles": [3, 31],
                    "flags": {"gap_fill": [False, True], "reuse_act_weight": [False, True],
                              "reuse_act_output": [False, True], "split_reduction": [False]}},
    "layer-b200": {"block_m": [16], "block_n": [64, 128], "block_k": [128], "k_split": [1], "consumer_warps": [8, 16, 30],
                   "n_stage": [4, 6], "prefetch_stride": [0, 3], "swizzles": [31],
                   "flags": {"gap_fill": [True], "reuse_act_weight": [False, True], "reuse_act_output": [False],
                             "split_reduction": [True]}},
    "defaults": {},
}


def graphs() -> dict:
    g = {"tiny-gemm": json.loads((FIX / "tiny-gemm.json").read_text()),
         "tiny-gemm-int4": json.loads((FIX / "tiny-gemm-int4.json").read_text()),
         "probe-layer": build_layer_graph(PROBE, 64),
         "probe-layer-int4": build_layer_graph(PROBE, 64, dtype="int4_w4a16"),
         "tiny-layer-lm": build_layer_graph(TINY, 48, lm_head=True)}
    return g


# (name, graph, hw, space, budget)
SEARCHES = [
    ("s01", "tiny-gemm", "l20", "tiny-full", 10000),
    ("s02", "tiny-gemm-int4", "l20", "tiny-full", 10000),
    ("s03", "tiny-gemm", "b200", "tiny-full", 10000),
    ("s04", "tiny-gemm", "l20", "tiny-full", 100),        # budget smaller than the kept set
    ("s05", "tiny-gemm", "l20", "tiny-full", 2400),       # budget runs out inside the improvement passes
    ("s06", "tiny-gemm", "l20", "defaults", 10000),
    ("s07", "probe-layer", "l20", "layer-small", 10000),
    ("s08", "probe-layer-int4", "l20", "layer-small", 40),
    ("s09", "probe-layer", "b200", "layer-b200", 10000),
    ("s10", "tiny-layer-lm", "b200", "layer-small", 24),
    ("s11", "probe-layer", "l20", "layer-a", 10000),      # slow in the reference (~2.5 min)
]


def run_cli(argv: list) -> tuple:
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            code = ref_cli.main(argv)
        except SystemExit as exc:  # argparse
            code = exc.code
    return code, out.getvalue(), err.getvalue()


def main() -> None:
    quick = "--quick" in sys.argv
    OUT.mkdir(parents=True, exist_ok=True)
    inputs = OUT / "inputs"
    inputs.mkdir(exist_ok=True)
    for name, g in graphs().items():
        (inputs / f"graph_{name}.json").write_text(json.dumps(g, indent=1) + "\n")
    for hw in ("l20", "b200"):
        (inputs / f"hw_{hw}.json").write_text((FIX / f"{hw}.json").read_text())
    for name, sp in SPACES.items():
        (inputs / f"space_{name}.json").write_text(json.dumps(sp) + "\n")

    manifest = {"searches": [], "cli": []}
    for name, g, hw, sp, budget in SEARCHES:
        if quick and name == "s11":
            continue
        t0 = time.time()
        argv = ["search", "--graph", str(inputs / f"graph_{g}.json"), "--hw", str(inputs / f"hw_{hw}.json"),
                "--space", str(inputs / f"space_{sp}.json"), "--budget", str(budget), "--threads", "4",
                "--out", str(OUT / f"{name}.trace")]
        code, out, err = run_cli(argv)
        (OUT / f"{name}.stdout").write_text(out)
        manifest["searches"].append({"name": name, "graph": g, "hw": hw, "space": sp, "budget": budget, "exit": code,
                                     "ref_seconds": round(time.time() - t0, 2)})
        print(name, code, f"{time.time() - t0:.1f}s", out.splitlines()[0] if out else err.strip()[:80], flush=True)

    # lower / dag / plan / simulate / validate / explain and the error paths
    gi = lambda n: str(inputs / f"graph_{n}.json")
    hi = lambda n: str(inputs / f"hw_{n}.json")
    si = lambda n: str(inputs / f"space_{n}.json")
    plan_a = {"tile": [16, 64, 64, 2], "n_stage": 2, "consumer_warps": 8, "prefetch_stride": 1, "swizzle": 31,
              "flags": {"gap_fill": True, "reuse_act_weight": True, "reuse_act_output": False, "split_reduction": False}}
    plan_b = {"tile": [16, 8, 16, 1], "n_stage": 2, "consumer_warps": 16, "swizzle": 0}
    plan_c = {"tile": [16, 64, 128, 1], "n_stage": 4, "consumer_warps": 16, "prefetch_stride": 2, "swizzle": 7,
              "flags": {"split_reduction": True, "reuse_act_output": True}}
    for n, p in (("a", plan_a), ("b", plan_b), ("c", plan_c)):
        (inputs / f"plan_{n}.json").write_text(json.dumps(p) + "\n")
    (inputs / "hw_unknown_field.json").write_text(json.dumps({"smem_max_bytes": 131072, "bogus": 1}) + "\n")
    (inputs / "hw_tiny_smem.json").write_text(json.dumps({"smem_max_bytes": 8192, "page_size_bytes": 4096}) + "\n")
    bad_trace = (OUT / "s01.trace").read_bytes().replace(b'"n_stage":3', b'"n_stage":2', 1)
    (inputs / "corrupt.trace").write_bytes(bad_trace)
    (inputs / "graph_forward_ref.json").write_text(json.dumps({
        "buffers": [{"id": "a", "space": "Global", "bytes": 64}, {"id": "b", "space": "Global", "bytes": 64}],
        "operators": [{"id": "o1", "kind": "RmsNorm", "dims": {"m": 1, "n": 8}, "inputs": ["b"], "outputs": ["a"]},
                      {"id": "o2", "kind": "RmsNorm", "dims": {"m": 1, "n": 8}, "inputs": ["a"], "outputs": ["b"]}]}))
    pi = lambda n: str(inputs / f"plan_{n}.json")
    cases = [
        ("lower_tiny", ["lower", "--graph", gi("tiny-gemm"), "--hw", hi("l20"), "--format", "json"]),
        ("lower_tiny_int4", ["lower", "--graph", gi("tiny-gemm-int4"), "--hw", hi("l20"), "--format", "json"]),
        ("lower_tiny_text", ["lower", "--graph", gi("tiny-gemm"), "--hw", hi("l20")]),
        ("lower_layer", ["lower", "--graph", gi("probe-layer"), "--hw", hi("l20"), "--space", si("layer-a"), "--format", "json"]),
        ("lower_layer_b200", ["lower", "--graph", gi("tiny-layer-lm"), "--hw", hi("b200"), "--space", si("layer-small"), "--format", "json"]),
        ("dag_tiny", ["dag", "--graph", gi("tiny-gemm"), "--hw", hi("l20")]),
        ("dag_layer", ["dag", "--graph", gi("probe-layer"), "--hw", hi("l20"), "--space", si("layer-a")]),
        ("dag_layer_int4", ["dag", "--graph", gi("probe-layer-int4"), "--hw", hi("l20"), "--space", si("layer-small")]),
        ("plan_tiny", ["plan", "--graph", gi("tiny-gemm"), "--hw", hi("l20"), "--space", si("tiny-full")]),
        ("plan_layer", ["plan", "--graph", gi("probe-layer"), "--hw", hi("b200"), "--space", si("layer-b200")]),
        ("sim_tiny_b", ["simulate", "--graph", gi("tiny-gemm"), "--hw", hi("l20"), "--plan", pi("b"), "--format", "json"]),
        ("sim_tiny_b_text", ["simulate", "--graph", gi("tiny-gemm"), "--hw", hi("l20"), "--plan", pi("b")]),
        ("sim_layer_a", ["simulate", "--graph", gi("probe-layer"), "--hw", hi("l20"), "--plan", pi("a"), "--format", "json"]),
        ("sim_layer_c", ["simulate", "--graph", gi("probe-layer"), "--hw", hi("b200"), "--plan", pi("c"), "--format", "json"]),
        ("sim_layer_int4_c", ["simulate", "--graph", gi("probe-layer-int4"), "--hw", hi("b200"), "--plan", pi("c"), "--format", "json"]),
        ("validate_a", ["validate", "--graph", gi("probe-layer"), "--hw", hi("l20"), "--plan", pi("a")]),
        ("explain_s01", ["explain", "--trace", str(OUT / "s01.trace"), "--graph", gi("tiny-gemm"), "--hw", hi("l20")]),
        ("explain_s07", ["explain", "--trace", str(OUT / "s07.trace"), "--graph", gi("probe-layer"), "--hw", hi("l20")]),
        ("err_missing_hw", ["lower", "--graph", gi("tiny-gemm")]),
        ("err_unknown_field", ["lower", "--graph", gi("tiny-gemm"), "--hw", str(inputs / "hw_unknown_field.json")]),
        ("err_no_feasible", ["search", "--graph", gi("tiny-gemm"), "--hw", str(inputs / "hw_tiny_smem.json"), "--space", si("tiny-full")]),
        ("err_corrupt_trace", ["explain", "--trace", str(inputs / "corrupt.trace"), "--graph", gi("tiny-gemm"), "--hw", hi("l20")]),
        ("err_forward_ref", ["lower", "--graph", str(inputs / "graph_forward_ref.json"), "--hw", hi("l20")]),
        ("err_wrong_graph", ["explain", "--trace", str(OUT / "s01.trace"), "--graph", gi("tiny-gemm-int4"), "--hw", hi("l20")]),
    ]
    timeline = OUT / "sim_layer_a.timeline.json"
    cases.append(("sim_layer_a_timeline", ["simulate", "--graph", gi("probe-layer"), "--hw", hi("l20"), "--plan", pi("a"),
                                           "--format", "json", "--timeline", str(timeline)]))
    for name, argv in cases:
        code, out, err = run_cli(argv)
        rel = [a.replace(str(OUT), "$G") for a in argv]
        (OUT / f"{name}.out").write_text(out)
        manifest["cli"].append({"name": name, "argv": rel, "exit": code, "stderr": err.replace(str(OUT), "$G")})
        print(name, code, len(out), flush=True)
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")


if __name__ == "__main__":
    main()
