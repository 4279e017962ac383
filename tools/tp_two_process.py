#!/usr/bin/env python
"""Tensor-parallel decode across PROCESSES: `tp` ranks, one process each, exchange the CUDA IPC handles of their
workspaces through torch.distributed (dist_utils.share_workspaces -- the start-up path the 8-GPU run takes) and then
publish their partial rows into each other's workspaces from inside the kernel.  With one GPU in the box the ranks
share it (148 // tp SMs each, gloo rendezvous; the driver time-slices the two contexts, so a step takes milliseconds):
this exercises the IPC mapping and the system-scope tagged-word exchange across address spaces, not performance.

    python tools/tp_two_process.py [tp] [steps]        (spawns the ranks itself)
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def rank_main(rank: int, tp: int, steps: int, port: int) -> None:
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(tp), LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import numpy as np
    import torch

    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200 import task_table as tt
    from paper_2605_11581_b200.dist_utils import RankGroup, share_workspaces
    from paper_2605_11581_b200.model_config import ModelConfig
    from paper_2605_11581_b200.plugin import MegaKernelPlugin, device_sm_count
    from paper_2605_11581_b200.weights import random_weights, rope_table

    n_gpus = torch.cuda.device_count()
    dev = rank % n_gpus                       # one GPU per rank when the box has them, else shared
    torch.cuda.set_device(dev)
    group = RankGroup(backend="gloo")         # NCCL refuses two ranks on one device; the handles are Python objects anyway
    cfg = ModelConfig(name="test-tp", hidden=512, n_layers=3, n_q_heads=8, n_kv_heads=2, head_dim=128,
                      intermediate=1536, vocab=3000, qkv_bias=True, qk_norm=False, tied_embed=True)
    max_ctx = 64
    w = random_weights(cfg, seed=0)
    sched = tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2, attn_min_chunk=16, l2_prefetch_kb=64)
    shared = n_gpus < tp
    n_sms = device_sm_count(dev) // (tp if shared else 1)
    pl = MegaKernelPlugin(cfg.shard(tp), sched, max_ctx=max_ctx, device=dev, n_sms=n_sms, tp_rank=rank, tp_size=tp)
    pl.bind_weights(w.shard(rank, tp))
    peers = share_workspaces(group, pl.workspace)
    assert len(peers) == tp and peers[rank].data_ptr() == pl.workspace.data_ptr()
    assert all(peers[r].numel() == pl.workspace.numel() for r in range(tp))
    pl.bind_peers(peers)
    torch.cuda.synchronize()
    group.barrier()
    g = torch.Generator().manual_seed(1)
    toks = torch.randint(0, cfg.vocab, (steps,), generator=g).tolist()
    ref = None
    if rank == 0:
        cos, sin = rope_table(cfg, max_ctx)
        ref = RefDecoder(cfg, w, max_ctx, cos, sin)
    vl = cfg.shard(tp).vocab
    worst = 0.0
    for pos, tok in enumerate(toks):
        out = pl.decode_step(tok, pos, want_logits=True)
        pl.check()
        mine = pl.logits[0, rank * vl:(rank + 1) * vl].cpu()
        parts = [None] * tp
        group.dist.all_gather_object(parts, (mine.numpy(), int(out.next_token.item())))
        assert len({p[1] for p in parts}) == 1, f"ranks disagree on the next token at step {pos}: {[p[1] for p in parts]}"
        if rank == 0:
            want = ref.step([tok], [pos])[0].numpy()
            got = np.concatenate([p[0] for p in parts])
            err = float(np.abs(got - want).max())
            worst = max(worst, err)
            assert err <= 2e-3, (pos, err)
            if np.sort(want)[-1] - np.sort(want)[-2] > 1e-2:
                assert parts[0][1] == int(want.argmax()), pos
    if rank == 0:
        print(f"tp_two_process ok: tp={tp} ranks in {tp} processes ({'one shared GPU' if shared else 'one GPU each'}), "
              f"{steps} steps, IPC-mapped workspaces, max |logit diff| vs oracle {worst:.2e}")
    group.barrier()
    pl.close()
    group.close()


if __name__ == "__main__":
    tp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.spawn(rank_main, args=(tp, steps, port), nprocs=tp, join=True)
