"""ModelConfig -> operator graph in the reference's JSON schema.

The reference ships no decoder-layer graph (SPEC.md names a
``qwen-decoder-layer.json`` fixture that is absent); this
builder emits one so the same file drives the reference planner and this one.
The layer is the twelve-operator chain of SURVEY.md appendix A

    norm1 qkv qk softmax pv oproj res1 norm2 upgate swiglu down res2 [+ final norm, lm_head]

using only the reference's eight operator kinds (``graph_ir.py:48-56``).  RoPE,
KV append, bias and QK-norm have no kind and move only a few KB, so they ride
inside the neighbouring operators of the kernel (csrc/adamk.cu) and do not
appear in the graph.

Activation buffers are sized for one ``block_m`` = 16-row padded tile
(``rows``).  Hidden-size vectors live in SharedPage space; intermediates wider
than ``wide_pages`` pages are declared Global, otherwise a full-size layer asks
for more resident pages than any SM has ("Resident
activation pages explode").
"""

from __future__ import annotations

import json

from ..model_config import ModelConfig

_ELEM = 2


def build_layer_graph(cfg: ModelConfig, ctx: int, *, rows: int = 16, m: int = 1, dtype: str = "fp16",
                      lm_head: bool = False, page_bytes: int = 16384, wide_pages: int = 2) -> dict:
    """One decoder layer (optionally followed by the final norm + LM head) as a graph dict."""
    h, i, d = cfg.hidden, cfg.intermediate, cfg.head_dim
    q_dim, qkv = cfg.q_dim, cfg.qkv_rows

    def act(cols: int) -> int:
        return rows * cols * _ELEM

    def space(cols: int) -> str:
        return "SharedPage" if act(cols) <= wide_pages * page_bytes else "Global"

    buffers = [
        ("x", space(h), act(h)), ("g1", "Global", h * _ELEM), ("xn", space(h), act(h)),
        ("wqkv", "Global", qkv * h * _ELEM), ("qkv", space(qkv), act(qkv)),
        ("kcache", "Global", cfg.n_kv_heads * ctx * d * _ELEM),
        ("scores", space(cfg.n_q_heads * ctx), act(cfg.n_q_heads * ctx)),
        ("probs", space(cfg.n_q_heads * ctx), act(cfg.n_q_heads * ctx)),
        ("vcache", "Global", cfg.n_kv_heads * ctx * d * _ELEM),
        ("attn", space(q_dim), act(q_dim)), ("wo", "Global", h * q_dim * _ELEM), ("o", space(h), act(h)),
        ("h1", space(h), act(h)), ("g2", "Global", h * _ELEM), ("h1n", space(h), act(h)),
        ("wug", "Global", 2 * i * h * _ELEM), ("ug", space(2 * i), act(2 * i)), ("act", space(i), act(i)),
        ("wd", "Global", h * i * _ELEM), ("d", space(h), act(h)), ("y", "Global", act(h)),
    ]

    def op(op_id, kind, n, k, inputs, outputs, weight=None, quant=False):
        return {"id": op_id, "kind": kind, "dims": {"m": m, "n": n, "k": k},
                "dtype": dtype if quant else "fp16", "inputs": inputs, "outputs": outputs, "weight": weight}

    operators = [
        op("norm1", "RmsNorm", h, 0, ["x"], ["xn"], "g1"),
        op("qkv", "Gemm", qkv, h, ["xn"], ["qkv"], "wqkv", quant=True),
        op("qk", "AttentionQK", ctx, d, ["qkv"], ["scores"], "kcache"),
        op("softmax", "Softmax", ctx, 0, ["scores"], ["probs"]),
        op("pv", "AttentionPV", d, ctx, ["probs"], ["attn"], "vcache"),
        op("oproj", "Gemm", h, q_dim, ["attn"], ["o"], "wo", quant=True),
        op("res1", "ResidualAdd", h, 0, ["o", "x"], ["h1"]),
        op("norm2", "RmsNorm", h, 0, ["h1"], ["h1n"], "g2"),
        op("upgate", "Gemm", 2 * i, h, ["h1n"], ["ug"], "wug", quant=True),
        op("swiglu", "Swiglu", i, 0, ["ug"], ["act"]),
        op("down", "Gemm", h, i, ["act"], ["d"], "wd", quant=True),
        op("res2", "ResidualAdd", h, 0, ["d", "h1"], ["y"]),
    ]
    if lm_head:
        buffers += [("gf", "Global", h * _ELEM), ("yn", space(h), act(h)),
                    ("wlm", "Global", cfg.vocab * h * _ELEM), ("logits", "Global", act(cfg.vocab))]
        operators += [op("normf", "RmsNorm", h, 0, ["y"], ["yn"], "gf"),
                      op("lm_head", "LmHead", cfg.vocab, h, ["yn"], ["logits"], "wlm", quant=True)]
    return {"buffers": [{"id": b, "space": s, "bytes": n} for b, s, n in buffers], "operators": operators}


def layer_graph_json(cfg: ModelConfig, ctx: int, **kw) -> str:
    return json.dumps(build_layer_graph(cfg, ctx, **kw), indent=1) + "\n"


def build_sm_slice_graph(cfg: ModelConfig, ctx: int, n_sms: int = 148, **kw) -> dict:
    """The share of one decoder layer that ONE SM executes in the decode MegaKernel: every GEMM keeps its full
    reduction dimension and 1/n_sms of its output rows (task_table.split_rows), attention covers one
    (q head, context chunk) unit.  The reference's planner models a single-SM pipeline ("no
    cross-SM/block scheduling"), so this -- not the whole layer -- is the graph whose schedule the kernel
    replays on each of its CTAs."""
    from dataclasses import replace

    def up(a: int, b: int) -> int:
        return -(-a // b)

    g = build_layer_graph(cfg, ctx, **kw)
    rows = {"qkv": up(cfg.qkv_rows, n_sms), "oproj": up(cfg.hidden, n_sms), "upgate": 2 * up(cfg.intermediate, n_sms),
            "down": up(cfg.hidden, n_sms)}
    chunk = max(8, up(ctx, max(1, n_sms // cfg.n_q_heads)))
    by_id = {o["id"]: o for o in g["operators"]}
    for oid, n in rows.items():
        by_id[oid]["dims"]["n"] = n
    by_id["swiglu"]["dims"]["n"] = rows["upgate"] // 2
    by_id["down"]["dims"]["k"] = cfg.intermediate
    by_id["qk"]["dims"]["n"] = chunk
    by_id["softmax"]["dims"]["n"] = chunk
    by_id["pv"]["dims"]["k"] = chunk
    del replace
    return g
