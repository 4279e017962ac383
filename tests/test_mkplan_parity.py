"""Bit-exact parity of paper_2605_11581_b200.mkplan with the reference planner.

Golden files under tests/golden/mkplan/ were produced by RUNNING the reference
(tools/make_mkplan_golden.py): solidified traces, DOT, lower summaries, simulation
reports, CLI text, stderr and exit codes.  Every test compares bytes."""

import contextlib
import io
import json
from pathlib import Path

import pytest

from conftest import GOLDEN
from paper_2605_11581_b200.mkplan import cli, search
from paper_2605_11581_b200.mkplan.graph_ir import load_graph
from paper_2605_11581_b200.mkplan.model_graph import build_layer_graph
from paper_2605_11581_b200.model_config import ModelConfig

G = GOLDEN / "mkplan"
MANIFEST = json.loads((G / "manifest.json").read_text()) if (G / "manifest.json").exists() else {"searches": [], "cli": []}


def _run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            code = cli.main(argv)
        except SystemExit as exc:
            code = exc.code
    return code, out.getvalue(), err.getvalue()


def test_manifest_present():
    assert len(MANIFEST["searches"]) >= 10 and len(MANIFEST["cli"]) >= 20


@pytest.mark.parametrize("case", MANIFEST["searches"], ids=lambda c: c["name"])
def test_search_trace_bytes_identical(case, tmp_path):
    if case.get("ref_seconds", 0) > 60:
        pytest.skip("covered by test_search_slow_case")
    _check_search(case, tmp_path)


@pytest.mark.slow
def test_search_slow_case(tmp_path):
    slow = [c for c in MANIFEST["searches"] if c.get("ref_seconds", 0) > 60]
    for case in slow:
        _check_search(case, tmp_path)


def _check_search(case, tmp_path):
    inp = G / "inputs"
    out_file = tmp_path / "t.trace"
    code, out, err = _run(["search", "--graph", str(inp / f"graph_{case['graph']}.json"),
                           "--hw", str(inp / f"hw_{case['hw']}.json"), "--space", str(inp / f"space_{case['space']}.json"),
                           "--budget", str(case["budget"]), "--threads", "1", "--out", str(out_file)])
    assert code == case["exit"], err
    assert out == (G / f"{case['name']}.stdout").read_text()
    assert out_file.read_bytes() == (G / f"{case['name']}.trace").read_bytes()


@pytest.mark.parametrize("case", MANIFEST["cli"], ids=lambda c: c["name"])
def test_cli_output_identical(case, tmp_path):
    argv = [a.replace("$G", str(G)) for a in case["argv"]]
    timeline = None
    if "--timeline" in argv:
        i = argv.index("--timeline")
        timeline = Path(argv[i + 1])
        argv[i + 1] = str(tmp_path / "timeline.json")
    code, out, err = _run(argv)
    assert code == case["exit"]
    assert out == (G / f"{case['name']}.out").read_text()
    assert err.replace(str(G), "$G") == case["stderr"]
    if timeline is not None:
        assert (tmp_path / "timeline.json").read_text() == timeline.read_text()


def test_threads_do_not_change_the_trace(tmp_path):
    inp = G / "inputs"
    texts = [(inp / "graph_tiny-gemm.json").read_text(), (inp / "hw_l20.json").read_text(),
             (inp / "space_tiny-full.json").read_text()]
    a = search.serialize_trace(search.run_search(*texts, budget=10000, parallel=1))
    b = search.serialize_trace(search.run_search(*texts, budget=10000, parallel=8))
    assert a == b == (G / "s01.trace").read_bytes()


@pytest.mark.parametrize("case", [c for c in MANIFEST["searches"] if c["name"] in ("s02", "s05", "s08")],
                         ids=lambda c: c["name"])
def test_worker_processes_do_not_change_the_trace(case, monkeypatch):
    """MK_PLANNER_PROCS: base simulations and improvement passes in forked workers (what makes a full-dimension
    search practical) -- the golden bytes at the golden budget, and the sequential bytes at budgets that run out inside
    the base simulations, between a gap fill and its role rebalance, and one short of everything."""
    inp = G / "inputs"
    texts = [(inp / f"graph_{case['graph']}.json").read_text(), (inp / f"hw_{case['hw']}.json").read_text(),
             (inp / f"space_{case['space']}.json").read_text()]
    monkeypatch.setenv("MK_PLANNER_PROCS", "3")
    full = search.run_search(*texts, budget=case["budget"])
    assert search.serialize_trace(full) == (G / f"{case['name']}.trace").read_bytes()
    kept, simulated = full.stats["kept"], full.stats["simulated"]
    for budget in sorted({max(1, kept // 2), kept + 1, kept + 2, kept + 7, max(1, simulated - 1)}):
        if budget >= case["budget"]:
            continue
        monkeypatch.setenv("MK_PLANNER_PROCS", "3")
        forked = search.serialize_trace(search.run_search(*texts, budget=budget))
        monkeypatch.setenv("MK_PLANNER_PROCS", "0")
        assert forked == search.serialize_trace(search.run_search(*texts, budget=budget, parallel=1)), budget


def test_round_trip_rebuild_and_compare():
    inp = G / "inputs"
    data = (G / "s07.trace").read_bytes()
    solid = search.parse_trace(data)
    assert search.serialize_trace(solid) == data
    cand, spec = search.rebuild_candidate(solid, (inp / "graph_probe-layer.json").read_text(),
                                          (inp / "hw_l20.json").read_text())
    assert [row[0] for row in solid.plan["programs"]["Consumer"]] == cand.role_programs[search.Role.Consumer]
    other = search.parse_trace((G / "s09.trace").read_bytes())
    diff = search.compare_traces(solid, other)
    assert "plan.n_stage" in diff and "score.makespan" in diff
    with pytest.raises(search.TraceFormatError):
        search.parse_trace(data.replace(b'"makespan":', b'"makespan": ', 1).replace(b"7", b"8", 1))


def test_appendix_a_graph_hash():
    """The ModelConfig -> graph builder reproduces SURVEY.md appendix A (graph_hash 4f249123...f881)."""
    probe = ModelConfig(name="probe-256", hidden=256, n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=64,
                        intermediate=512, vocab=1024)
    g = load_graph(json.dumps(build_layer_graph(probe, 64)))
    assert search.content_hash(g.canonical_dict()) == "4f24912339cce61feb64a56e515aa990ab8ff56f19eed3693ef5fcc7fa18f881"
