"""Parity of the CUDA MegaKernel (through the C ABI) against the CPU oracle.

Every test here needs a B200 (``-m gpu``).  Tolerances: fp32 activations on both
sides, so the only difference is summation order -> logits max-abs <= 2e-3 here
(north-star bound: 2e-2, cosine >= 0.9995), greedy tokens identical, packed
weights and KV cache bit-exact / within one bf16 ulp.
"""

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import TINY, TINY_QWEN3, ModelConfig

pytestmark = pytest.mark.gpu

D128 = ModelConfig(name="test-d128", hidden=512, n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=128,
                   intermediate=1280, vocab=4096)
D128_Q3 = ModelConfig(name="test-d128-q3", hidden=512, n_layers=3, n_q_heads=8, n_kv_heads=2, head_dim=128,
                      intermediate=1536, vocab=3000, qkv_bias=False, qk_norm=True, tied_embed=False)

SCHEDS = {
    "c8": tt.KernelSchedule(consumer_warps=8, n_stage=4, rows_per_tile=16, ktile_chunks=2, attn_min_chunk=8),
    "c4": tt.KernelSchedule(consumer_warps=4, n_stage=3, rows_per_tile=16, ktile_chunks=1, attn_min_chunk=16),
    "c16": tt.KernelSchedule(consumer_warps=16, n_stage=5, rows_per_tile=32, ktile_chunks=2, attn_min_chunk=8),
    # the profiled default shape (7 consumer warps + Loader = 8 warps, 56 KB slots) with L2 prefetch and an in-flight cap
    "c7": tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2, attn_min_chunk=16,
                            l2_prefetch_kb=64, inflight=2),
    # small ring slots: the down projection spans several k-tiles, so its input vector is streamed in with
    # cp.async (down_streamed), including a zero-padded last chunk for the tiny models (I = 704)
    "c7s": tt.KernelSchedule(consumer_warps=7, n_stage=6, rows_per_tile=14, ktile_chunks=1, attn_min_chunk=16),
    "c7m": tt.KernelSchedule(consumer_warps=7, n_stage=6, rows_per_tile=28, ktile_chunks=1, attn_min_chunk=16,
                             l2_prefetch_kb=32),
    "c7m_nostream": tt.KernelSchedule(consumer_warps=7, n_stage=6, rows_per_tile=28, ktile_chunks=1, attn_min_chunk=16,
                                      stream_down=False),
    # fused down projection: gate/up keeps its SwiGLU outputs on the SM, multiplies its own K-slice of the down
    # projection (T_DOWNK) and the partial rows are summed by T_HRED tasks
    "c7f": tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2, attn_min_chunk=16,
                             l2_prefetch_kb=64, inflight=2, fuse_down=True),
    "c8f": tt.KernelSchedule(consumer_warps=8, n_stage=4, rows_per_tile=16, ktile_chunks=2, attn_min_chunk=8, fuse_down=True),
    "c4f": tt.KernelSchedule(consumer_warps=4, n_stage=3, rows_per_tile=16, ktile_chunks=1, attn_min_chunk=16, fuse_down=True),
}


def _setup(cfg, sched, max_ctx=128, seed=0):
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.plugin import MegaKernelPlugin
    from paper_2605_11581_b200.weights import random_weights, rope_table

    w = random_weights(cfg, seed=seed)
    cos, sin = rope_table(cfg, max_ctx)
    ref = RefDecoder(cfg, w, max_ctx, cos, sin)
    plug = MegaKernelPlugin(cfg, sched, max_ctx=max_ctx)
    plug.bind_weights(w)
    return w, ref, plug


def _cos(a, b):
    return float((a * b).sum() / (np.linalg.norm(a) * np.linalg.norm(b)))


@pytest.mark.parametrize("cfg,sname", [(TINY, "c8"), (TINY_QWEN3, "c8"), (D128, "c8"), (D128_Q3, "c8"),
                                       (TINY, "c4"), (D128, "c16"), (D128, "c7"), (D128_Q3, "c7"), (TINY_QWEN3, "c7"),
                                       (TINY, "c7s"), (TINY_QWEN3, "c7s"), (D128, "c7m"), (D128_Q3, "c7m"),
                                       (D128, "c7m_nostream"), (TINY, "c7f"), (TINY_QWEN3, "c8f"), (D128, "c7f"),
                                       (D128_Q3, "c7f"), (D128_Q3, "c4f")],
                         ids=lambda v: v if isinstance(v, str) else v.name)
def test_stepwise_logits_match_oracle(cfg, sname):
    """Teacher-forced: 40 steps (crossing the single-chunk -> split-KV boundary),
    per-step logits, greedy token and the KV cache rows against the oracle."""
    w, ref, plug = _setup(cfg, SCHEDS[sname])
    g = torch.Generator().manual_seed(1)
    toks = torch.randint(0, cfg.vocab, (40,), generator=g).tolist()
    worst = 0.0
    for pos, tok in enumerate(toks):
        want = ref.step([tok], [pos])[0].numpy()
        out = plug.decode_step(tok, pos, want_logits=True)
        plug.check()
        got = out.logits[0].cpu().numpy()
        err = float(np.abs(got - want).max())
        worst = max(worst, err)
        assert err <= 2e-3, (pos, err)
        assert _cos(got, want) >= 0.9995
        srt = np.sort(want)
        if srt[-1] - srt[-2] > 1e-2:
            assert int(out.next_token.item()) == int(want.argmax()), pos
    kc, vc = plug.kv_view()
    np.testing.assert_allclose(kc[:, 0, :, :40].float().cpu().numpy(), ref.k_cache[:, 0, :, :40].float().numpy(),
                               atol=4e-2, rtol=1e-2)
    np.testing.assert_allclose(vc[:, 0, :, :40].float().cpu().numpy(), ref.v_cache[:, 0, :, :40].float().numpy(),
                               atol=4e-2, rtol=1e-2)
    plug.close()


@pytest.mark.parametrize("cfg,sname", [(TINY, "c8"), (D128_Q3, "c8"), (D128_Q3, "c7f")], ids=lambda v: v if isinstance(v, str) else v.name)
def test_device_packer_is_bit_exact(cfg, sname):
    w, _, plug = _setup(cfg, SCHEDS[sname])
    want = tt.pack_weights_reference(plug.table, w)
    got = plug.packed[:plug.table.packed_weight_bytes].cpu().numpy().view(np.uint16)
    assert (got == want).all()
    plug.close()


@pytest.mark.parametrize("cfg", [TINY, TINY_QWEN3], ids=lambda c: c.name)
def test_matches_hf_golden_teacher_forced(cfg):
    """BASELINE.json configs[0] against the Hugging Face golden vectors: 16-token
    prompt, then the 32 golden tokens fed back; logits within the north-star
    tolerance at every step, argmax equal wherever HF's own margin is not a near-tie."""
    gold = np.load(GOLDEN / f"decode_{cfg.name}.npz")
    _, ref, plug = _setup(cfg, SCHEDS["c8"])
    prompt, gtoks = gold["prompt"].tolist(), gold["tokens"].tolist()
    for pos, tok in enumerate(prompt[:-1]):
        plug.decode_step(tok, pos, want_logits=False)
    feed = [prompt[-1]] + gtoks[:-1]
    srt = np.sort(gold["logits"], axis=1)
    margin = srt[:, -1] - srt[:, -2]
    checked = 0
    for i, tok in enumerate(feed):
        out = plug.decode_step(tok, len(prompt) - 1 + i, want_logits=True)
        plug.check()
        got = out.logits[0].cpu().numpy()
        assert np.abs(got - gold["logits"][i]).max() <= 2e-2, i
        assert _cos(got, gold["logits"][i]) >= 0.9995
        if margin[i] > 4e-2:
            assert int(out.next_token.item()) == gtoks[i], i
            checked += 1
    assert checked >= 16
    plug.close()


@pytest.mark.parametrize("cfg", [TINY, D128_Q3], ids=lambda c: c.name)
def test_device_resident_greedy_loop_matches_oracle(cfg):
    """64 free-running greedy steps with no host round trip (auto_advance) produce
    the oracle's token sequence (north star: identical over the first 64 steps)."""
    _, ref, plug = _setup(cfg, SCHEDS["c8"])
    g = torch.Generator().manual_seed(5)
    prompt = torch.randint(0, cfg.vocab, (16,), generator=g).tolist()
    want, want_logits = ref.generate(prompt, 64, stepwise_prefill=True)
    for pos, tok in enumerate(prompt[:-1]):
        plug.decode_step(tok, pos, want_logits=False)
    plug.set_state(prompt[-1], len(prompt) - 1)
    toks = []
    for _ in range(64):
        plug.enqueue(want_logits=False, auto_advance=True)
        toks.append(plug.next_token.clone())
    plug.check()
    got = [int(t.item()) for t in toks]
    srt = torch.stack(want_logits).sort(dim=1).values
    margin = (srt[:, -1] - srt[:, -2]).numpy()
    first_tie = int(np.argmax(margin < 1e-4)) if (margin < 1e-4).any() else 64
    assert got[:first_tie] == want[:first_tie]
    assert first_tie >= 32, f"near-tie at step {first_tie}; pick another seed"
    assert int(plug.positions.item()) == len(prompt) - 1 + 64
    plug.close()


def test_host_buffer_step_equals_the_device_resident_loop():
    """`adamk_decode_step_host` (host token / position in, host next token out, one C call per token) produces the
    token sequence of the device-resident loop, and reports bad arguments."""
    cfg = TINY
    _, ref, plug = _setup(cfg, SCHEDS["c7"])
    g = torch.Generator().manual_seed(5)
    prompt = torch.randint(0, cfg.vocab, (16,), generator=g).tolist()
    for pos, tok in enumerate(prompt[:-1]):
        plug.decode_step(tok, pos, want_logits=False)
    plug.set_state(prompt[-1], len(prompt) - 1)
    dev = []
    for _ in range(24):
        plug.enqueue(want_logits=False, auto_advance=True)
        dev.append(plug.next_token.clone())
    plug.check()
    dev = [int(t.item()) for t in dev]
    tok, pos, host = prompt[-1], len(prompt) - 1, []
    for _ in range(24):
        tok = plug.decode_step_host(tok, pos)
        pos += 1
        host.append(tok)
    assert host == dev
    assert int(plug.next_token.item()) == host[-1] and int(plug.positions.item()) == pos - 1
    plug.close()
    from paper_2605_11581_b200.plugin import AdamkError, MegaKernelPlugin
    unbound = MegaKernelPlugin(TINY, SCHEDS["c7"], max_ctx=64)
    with pytest.raises(AdamkError):          # step before bind_weights
        unbound.decode_step_host(1, 0)
    unbound.close()


@pytest.mark.parametrize("sname", ["c8", "c7"])
def test_long_context_split_kv(sname):
    """Context 700 with a small min chunk -> every chunk slot active, multi-block units, multi-record merge."""
    cfg = D128
    w, ref, plug = _setup(cfg, SCHEDS[sname], max_ctx=1024)
    g = torch.Generator().manual_seed(2)
    prompt = torch.randint(0, cfg.vocab, (700,), generator=g).tolist()
    ref.prefill(prompt)
    kc, vc = plug.kv_view()
    kc[:, 0, :, :700] = ref.k_cache[:, 0, :, :700].to(kc.device)
    vc[:, 0, :, :700] = ref.v_cache[:, 0, :, :700].to(vc.device)
    tok = 17
    for pos in range(700, 704):
        want = ref.step([tok], [pos])[0].numpy()
        out = plug.decode_step(tok, pos)
        plug.check()
        got = out.logits[0].cpu().numpy()
        assert np.abs(got - want).max() <= 2e-3
        tok = int(want.argmax())
        assert int(out.next_token.item()) == tok
    plug.close()


def test_error_paths():
    from paper_2605_11581_b200.plugin import AdamkError, MegaKernelPlugin

    plug = MegaKernelPlugin(TINY, SCHEDS["c8"], max_ctx=64)
    with pytest.raises(AdamkError):          # step before bind_weights
        plug.decode_step(1, 0)
    plug.close()


def test_host_step_refuses_inputs_that_would_trap():
    """`adamk_decode_step_host` validates the host token / position before copying or launching: a position at max_ctx
    or a token outside the vocabulary is an AdamkError (ADAMK_E_INVALID), the CUDA context and the handle stay usable
    and the next good step gives the oracle's logits (on the device the same input traps)."""
    from paper_2605_11581_b200.plugin import AdamkError

    cfg, max_ctx = TINY, 24
    _, ref, plug = _setup(cfg, SCHEDS["c7f"], max_ctx=max_ctx)
    g = torch.Generator().manual_seed(9)
    prompt = torch.randint(0, cfg.vocab, (8,), generator=g).tolist()
    for pos, tok in enumerate(prompt):
        got = plug.decode_step_host(tok, pos, want_logits=True)
        want = ref.step(tok, pos)
        for bad_tok, bad_pos in ((tok, max_ctx), (tok, -1), (cfg.vocab, pos), (-2, pos)):
            with pytest.raises(AdamkError):
                plug.decode_step_host(bad_tok, bad_pos)
    plug.check()
    assert got == int(want.argmax())
    np.testing.assert_allclose(plug.logits.cpu().numpy().reshape(-1), want.numpy().reshape(-1), atol=2e-3, rtol=0)
    plug.close()


def test_hybrid_engine_generate_matches_oracle():
    """Engine hook: prefill (decode-path backend) then a device-resident decode loop."""
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.engine import HybridEngine
    from paper_2605_11581_b200.weights import random_weights, rope_table

    cfg = D128
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, 128)
    ref = RefDecoder(cfg, w, 128, cos, sin)
    g = torch.Generator().manual_seed(7)
    prompt = torch.randint(0, cfg.vocab, (24,), generator=g).tolist()
    want, logits = ref.generate(prompt, 24, stepwise_prefill=True)
    eng = HybridEngine(cfg, w, max_ctx=128, schedule=SCHEDS["c8"], prefill_backend="decode")
    res = eng.generate(prompt, 24)
    srt = torch.stack(logits).sort(dim=1).values
    margin = (srt[:, -1] - srt[:, -2]).numpy()
    first_tie = int(np.argmax(margin < 1e-4)) if (margin < 1e-4).any() else 24
    assert res.tokens[:first_tie] == want[:first_tie] and first_tie >= 12
    assert res.prefill_launches == 23 and res.decode_launches == 24
    eng.close()


def test_default_schedule_runs_and_matches_oracle():
    """The shipped default schedule (schedules.default_schedule) on a mid-size model: logits parity over
    a few steps that start inside a prefilled context."""
    from paper_2605_11581_b200.schedules import default_schedule

    cfg = D128_Q3
    w, ref, plug = _setup(cfg, default_schedule(cfg), max_ctx=512)
    g = torch.Generator().manual_seed(11)
    prompt = torch.randint(0, cfg.vocab, (300,), generator=g).tolist()
    ref.prefill(prompt)
    kc, vc = plug.kv_view()
    kc[:, 0, :, :300] = ref.k_cache[:, 0, :, :300].to(kc.device)
    vc[:, 0, :, :300] = ref.v_cache[:, 0, :, :300].to(vc.device)
    tok = 5
    for pos in range(300, 306):
        want = ref.step([tok], [pos])[0].numpy()
        out = plug.decode_step(tok, pos)
        plug.check()
        got = out.logits[0].cpu().numpy()
        assert np.abs(got - want).max() <= 2e-3
        tok = int(want.argmax())
    plug.close()


def test_repeated_runs_are_bitwise_reproducible():
    """The tagged-word exchange sums in a fixed order: two runs of the same steps give identical logits."""
    cfg = D128
    outs = []
    for _ in range(2):
        _, _, plug = _setup(cfg, SCHEDS["c7"])
        acc = []
        for pos, tok in enumerate([3, 17, 4000, 25, 999, 1, 2, 3]):
            acc.append(plug.decode_step(tok, pos).logits[0].clone())
        plug.check()
        outs.append(torch.stack(acc).cpu())
        plug.close()
    assert torch.equal(outs[0], outs[1])


def test_tensor_parallel_across_processes_with_ipc_workspaces():
    """The start-up path of a multi-GPU tensor-parallel run, on hardware: two PROCESSES exchange the CUDA IPC handles
    of their workspaces through torch.distributed (dist_utils.share_workspaces), map each other's buffers and then
    publish partial rows into them from inside the kernel (system-scope tagged words across address spaces).  With one
    GPU in the box the ranks share it (74 SMs each; the two contexts are time-sliced).  Logits are checked against the
    unsharded oracle and the ranks must agree on every token (tools/tp_two_process.py)."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    res = subprocess.run([sys.executable, str(root / "tools" / "tp_two_process.py"), "2", "4"],
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "tp_two_process ok: tp=2 ranks in 2 processes" in res.stdout


@pytest.mark.parametrize("tp", [2, 4])
def test_tensor_parallel_ranks_on_one_gpu(tp):
    """In-kernel tensor parallelism (adamk.cu: tp_publish / ll_gather_tp / tp_argmax_exchange): `tp` ranks with
    148 // tp SMs each run concurrently on one GPU and store their partial O-proj / down-proj rows and LM-head
    argmax into each other's workspaces, as ranks on different GPUs do through peer-mapped memory.  Logits and
    tokens are checked against the unsharded oracle inside tools/tp_single_gpu.py; it runs in a subprocess so a
    device trap (watchdog) cannot poison this process."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    res = subprocess.run([sys.executable, str(root / "tools" / "tp_single_gpu.py"), str(tp), "16"],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert f"tp={tp} on one GPU" in res.stdout and "steps ok" in res.stdout


def test_tp_requires_peers():
    from paper_2605_11581_b200.plugin import AdamkError, MegaKernelPlugin
    from paper_2605_11581_b200.weights import random_weights

    cfg = D128_Q3
    plug = MegaKernelPlugin(cfg.shard(2), SCHEDS["c7"], max_ctx=64, n_sms=74, tp_rank=1, tp_size=2)
    plug.bind_weights(random_weights(cfg, seed=0).shard(1, 2))
    with pytest.raises(AdamkError):          # step before bind_peers
        plug.decode_step(1, 0)
    with pytest.raises(AdamkError):          # peer list of the wrong length
        plug.bind_peers([plug.workspace])
    plug.close()


@pytest.mark.parametrize("batch", [2, 4])
def test_batch_lanes_match_oracle(batch):
    """BASELINE.json configs[2] (batch sweep), CUDA-core path: `batch` sequences at different positions, each on
    its own SM partition, all streaming one packed weight buffer; per-sequence logits / tokens vs the oracle."""
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.plugin import BatchLanes
    from paper_2605_11581_b200.weights import random_weights, rope_table

    cfg = D128_Q3
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, 128)
    refs = [RefDecoder(cfg, w, 128, cos, sin) for _ in range(batch)]
    lanes = BatchLanes(cfg, SCHEDS["c7"], max_ctx=128, batch=batch)
    lanes.bind_weights(w)
    assert all(lane.packed.data_ptr() == lanes.lanes[0].packed.data_ptr() for lane in lanes.lanes)
    g = torch.Generator().manual_seed(9)
    # sequence b starts b * 3 tokens later: the lanes run at different positions in the same step
    seqs = [torch.randint(0, cfg.vocab, (20,), generator=g).tolist() for _ in range(batch)]
    pos = [0] * batch
    for step in range(20 + 3 * (batch - 1)):
        live = [b for b in range(batch) if 0 <= step - 3 * b < 20]
        toks = [seqs[b][step - 3 * b] if b in live else 0 for b in range(batch)]
        # idle lanes re-run position 0 with token 0 (harmless: their cache row 0 is rewritten when they go live)
        out = lanes.decode_step(toks, [pos[b] if b in live else 0 for b in range(batch)])
        lanes.check()
        for b in live:
            want = refs[b].step([toks[b]], [pos[b]])[0].numpy()
            got = out.logits[b].cpu().numpy()
            assert np.abs(got - want).max() <= 2e-3, (step, b)
            if np.sort(want)[-1] - np.sort(want)[-2] > 1e-2:
                assert int(out.next_token[b].item()) == int(want.argmax())
            pos[b] += 1
    lanes.close()


def test_plugin_from_searched_trace_matches_oracle():
    """The drop-in flow end to end: mkplan search (SM-slice graph, b200.json) -> SolidifiedTrace bytes ->
    MegaKernelPlugin.from_trace -> decode steps that match the oracle."""
    import json
    from pathlib import Path

    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.mkplan import model_graph, search
    from paper_2605_11581_b200.plugin import MegaKernelPlugin
    from paper_2605_11581_b200.weights import random_weights, rope_table

    cfg = TINY
    graph = model_graph.build_sm_slice_graph(cfg, 64, n_sms=148)
    hw = (Path(tt.__file__).parent / "mkplan" / "fixtures" / "b200.json").read_text()
    space = {"block_m": [16], "block_n": [16, 32], "block_k": [256], "k_split": [1], "consumer_warps": [4, 8],
             "n_stage": [2, 3], "prefetch_stride": [1], "swizzles": [31]}
    text = search.serialize_trace(search.run_search(json.dumps(graph), hw, json.dumps(space), 100))
    plug = MegaKernelPlugin.from_trace(cfg, text, max_ctx=64, attn_min_chunk=16)
    w = random_weights(cfg, seed=0)
    plug.bind_weights(w)
    cos, sin = rope_table(cfg, 64)
    ref = RefDecoder(cfg, w, 64, cos, sin)
    for pos, tok in enumerate([7, 300, 12, 999, 4, 4, 250, 31]):
        want = ref.step([tok], [pos])[0].numpy()
        got = plug.decode_step(tok, pos).logits[0].cpu().numpy()
        plug.check()
        assert np.abs(got - want).max() <= 2e-3
    plug.close()


def test_streamed_down_projection_is_used_and_bit_identical():
    """The schedules above really take the streamed path (several k-tiles for the down projection), and the
    streamed and the up-front gather give bit-identical logits (same values, same summation order)."""
    cfg = D128
    t = tt.build_task_table(cfg, SCHEDS["c7m"], n_sms=148)
    down = t.tasks[t.tasks[:, tt.F_TYPE] == tt.T_DOWN]
    assert (down[:, tt.F_NKTILES] > 1).all() and (down[:, tt.F_NTILES] == 1).all()
    outs = []
    for name in ("c7m", "c7m_nostream"):
        _, _, plug = _setup(cfg, SCHEDS[name])
        acc = [plug.decode_step(tok, pos).logits[0].clone() for pos, tok in enumerate([3, 17, 4000, 25, 999, 1])]
        plug.check()
        outs.append(torch.stack(acc).cpu())
        plug.close()
    assert torch.equal(outs[0], outs[1])


def test_full_size_qwen25_1p5b_matches_oracle():
    """BASELINE.json configs[1] at full size, the shipped default schedule: a 96-token context prefilled by the
    oracle, then decode steps whose logits (151 936 of them) and greedy tokens are compared with the CPU oracle.
    Tolerance as for the small models: fp32 everywhere, so only the summation order differs."""
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.model_config import QWEN25_1P5B
    from paper_2605_11581_b200.plugin import MegaKernelPlugin
    from paper_2605_11581_b200.schedules import default_schedule
    from paper_2605_11581_b200.weights import random_weights, rope_table

    cfg = QWEN25_1P5B
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, 128)
    ref = RefDecoder(cfg, w, 128, cos, sin)
    plug = MegaKernelPlugin(cfg, default_schedule(cfg), max_ctx=128)
    plug.bind_weights(w)
    g = torch.Generator().manual_seed(1)
    prompt = torch.randint(0, cfg.vocab, (96,), generator=g).tolist()
    ref.prefill(prompt)
    kc, vc = plug.kv_view()
    kc[:, 0, :, :96] = ref.k_cache[:, 0, :, :96].to(kc.device)
    vc[:, 0, :, :96] = ref.v_cache[:, 0, :, :96].to(vc.device)
    tok = 11
    for pos in range(96, 100):
        want = ref.step([tok], [pos])[0].numpy()
        out = plug.decode_step(tok, pos)
        plug.check()
        got = out.logits[0].cpu().numpy()
        assert np.abs(got - want).max() <= 2e-3, float(np.abs(got - want).max())
        assert _cos(got, want) >= 0.9995
        srt = np.sort(want)
        tok = int(want.argmax())
        if srt[-1] - srt[-2] > 1e-2:
            assert int(out.next_token.item()) == tok
    plug.close()


def test_qwen25_1p5b_greedy_64_tokens_identical():
    """North-star criterion on BASELINE.json configs[1]: after the 512-token prompt of bench.py, 64 free-running
    greedy steps of the kernel (device-resident loop, one launch per token) emit the oracle's tokens -- all 64, no
    near-tie escape: the prompt seed is chosen so that the oracle's own top-1 / top-2 margin never comes near the logit
    tolerance (the minimum margin is printed)."""
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.model_config import QWEN25_1P5B
    from paper_2605_11581_b200.plugin import MegaKernelPlugin
    from paper_2605_11581_b200.schedules import default_schedule
    from paper_2605_11581_b200.weights import random_weights, rope_table

    cfg = QWEN25_1P5B
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, 640)
    ref = RefDecoder(cfg, w, 640, cos, sin)
    # prompt seed 3: the oracle's own top-1 / top-2 margin stays >= 1.0e-2 over all 64 steps (seeds 1..8 scanned on the
    # CPU oracle; 1, 2 and 4 dip below 5e-3) -- five times the 2e-3 logit tolerance
    g = torch.Generator().manual_seed(3)
    prompt = torch.randint(0, cfg.vocab, (512,), generator=g).tolist()
    logits = ref.prefill(prompt)
    plug = MegaKernelPlugin(cfg, default_schedule(cfg), max_ctx=640)
    plug.bind_weights(w)
    kc, vc = plug.kv_view()
    kc[:, 0, :, :512] = ref.k_cache[:, 0, :, :512].to(kc.device)
    vc[:, 0, :, :512] = ref.v_cache[:, 0, :, :512].to(vc.device)
    first = int(torch.argmax(logits))
    want, margins = [], []
    tok, pos = first, 512
    for _ in range(64):
        lg = ref.step([tok], [pos])[0]
        top = torch.topk(lg, 2).values
        margins.append(float(top[0] - top[1]))
        tok = int(torch.argmax(lg))
        want.append(tok)
        pos += 1
    plug.set_state(first, 512)
    outs = []
    for _ in range(64):
        plug.enqueue(want_logits=False, auto_advance=True)
        outs.append(plug.next_token.clone())
    plug.check()
    got = [int(t.item()) for t in outs]
    margins = np.asarray(margins)
    print(f"greedy 64: minimum top-1/top-2 margin of the oracle {margins.min():.2e} at step {int(margins.argmin())}")
    assert margins.min() >= 5e-3, "the documented prompt seed no longer keeps the margins clear of the tolerance"
    assert got == want
    plug.close()


def test_hybrid_engine_library_prefill_matches_oracle():
    """Engine hook with the library prefill backend (prefill on the serving engine's own operators,
    decode on the MegaKernel): fp32 library GEMMs fill the plugin's KV cache, the first generated token already
    comes from a MegaKernel launch, and the greedy continuation matches the oracle."""
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.engine import HybridEngine
    from paper_2605_11581_b200.weights import random_weights, rope_table

    cfg = D128_Q3
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, 256)
    ref = RefDecoder(cfg, w, 256, cos, sin)
    g = torch.Generator().manual_seed(7)
    prompt = torch.randint(0, cfg.vocab, (150,), generator=g).tolist()
    want, logits = ref.generate(prompt, 24)
    eng = HybridEngine(cfg, w, max_ctx=256, schedule=SCHEDS["c7"], prefill_backend="library")
    res = eng.generate(prompt, 24)
    kc, _ = eng.plugin.kv_view()
    np.testing.assert_allclose(kc[:, 0, :, :149].float().cpu().numpy(), ref.k_cache[:, 0, :, :149].float().numpy(),
                               atol=4e-2, rtol=1e-2)
    srt = torch.stack(logits).sort(dim=1).values
    margin = (srt[:, -1] - srt[:, -2]).numpy()
    first_tie = int(np.argmax(margin < 1e-3)) if (margin < 1e-3).any() else 24
    assert res.tokens[:first_tie] == want[:first_tie] and first_tie >= 12
    assert res.prefill_launches == 0 and res.decode_launches == 24
    eng.close()


def test_full_size_qwen3_8b_matches_oracle_tp1_and_tp2():
    """BASELINE.json configs[3] at full size (Qwen3-8B: H 4096, 32/8 heads, I 12288, QK-norm, untied 151 936-row LM
    head, 36 layers, 15 GB of weights): per-step logits of the MegaKernel against the CPU oracle, first as one rank
    with all 148 SMs (the fused down projection: three 256-row blocks per warp), then as two tensor-parallel ranks of
    74 SMs each on the one GPU (heads / intermediate / vocabulary split, in-kernel partial-row exchange).

    Tolerance: the north star's (max-abs 2e-2, cosine 0.9995).  Both sides keep fp32 activations, but the KV cache is
    bf16 on both: with 1024 V elements per layer a few land within one fp32 ulp of a bf16 rounding boundary, the two
    summation orders round them to neighbouring bf16 values (measured: one 7.8e-3 flip in layer 0), and 36 layers
    carry that to ~1e-2 in the logits -- fused and unfused schedules give the same numbers (tools/dbg_8b.py)."""
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.model_config import QWEN3_8B
    from paper_2605_11581_b200.plugin import MegaKernelPlugin, device_sm_count
    from paper_2605_11581_b200.schedules import default_schedule
    from paper_2605_11581_b200.weights import random_weights, rope_table

    cfg, max_ctx, steps = QWEN3_8B, 32, 4
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, max_ctx)
    ref = RefDecoder(cfg, w, max_ctx, cos, sin)
    g = torch.Generator().manual_seed(1)
    toks = torch.randint(0, cfg.vocab, (steps,), generator=g).tolist()
    wants = [ref.step([tok], [pos])[0].numpy() for pos, tok in enumerate(toks)]
    del ref

    from dataclasses import replace

    from paper_2605_11581_b200.schedules import fit_schedule

    default = default_schedule(cfg)
    assert not default.fuse_down          # three 256-row blocks per warp: the default keeps the row-split down projection
    fused = fit_schedule(cfg, replace(default, fuse_down=True, inflight=0), keep_fused=True)
    assert fused.fuse_down
    for label, sched in (("default", default), ("fused down projection", fused)):
        plug = MegaKernelPlugin(cfg, sched, max_ctx=max_ctx)
        plug.bind_weights(w)
        for pos, tok in enumerate(toks):
            out = plug.decode_step(tok, pos, want_logits=True)
            plug.check()
            got = out.logits[0].cpu().numpy()
            err = float(np.abs(got - wants[pos]).max())
            assert err <= 2e-2, (label, pos, err)
            assert _cos(got, wants[pos]) >= 0.9995
            srt = np.sort(wants[pos])
            if srt[-1] - srt[-2] > 5e-2:
                assert int(out.next_token.item()) == int(wants[pos].argmax())
            print(f"qwen3-8b tp=1 ({label}) step {pos}: max |logit diff| {err:.2e}")
        plug.close()
        del plug
        torch.cuda.empty_cache()

    tp = 2
    lcfg = cfg.shard(tp)
    n_sms = device_sm_count(0) // tp
    sched2 = default_schedule(lcfg, n_sms=n_sms, tp_size=tp)
    plugs, streams = [], []
    for r in range(tp):
        pl = MegaKernelPlugin(lcfg, sched2, max_ctx=max_ctx, n_sms=n_sms, tp_rank=r, tp_size=tp)
        pl.bind_weights(w.shard(r, tp))
        plugs.append(pl)
        streams.append(torch.cuda.Stream())
    for pl in plugs:
        pl.bind_peers([q.workspace for q in plugs])
    torch.cuda.synchronize()
    vl = lcfg.vocab
    for pos, tok in enumerate(toks):
        outs = []
        for r, pl in enumerate(plugs):
            with torch.cuda.stream(streams[r]):
                outs.append(pl.decode_step(tok, pos, want_logits=True))
        for pl in plugs:
            pl.check()
        got = np.concatenate([plugs[r].logits[0, r * vl:(r + 1) * vl].cpu().numpy() for r in range(tp)])
        err = float(np.abs(got - wants[pos]).max())
        assert err <= 2e-2, (pos, err)
        assert _cos(got, wants[pos]) >= 0.9995
        assert int(outs[0].next_token.item()) == int(outs[1].next_token.item())
        print(f"qwen3-8b tp=2 step {pos}: max |logit diff| {err:.2e}")
    for pl in plugs:
        pl.close()
