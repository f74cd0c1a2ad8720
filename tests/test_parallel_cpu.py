"""N>1 host logic on CPU with gloo, world size 2: sequence partition,
shard-order all-gather, the global-head-order EMA input (bit-exact vs one process) and
the vocab-sharded confidence merge (vs the unsharded confidence)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import confkv_oracle as O
from oracle import scenarios as S
from paper_2605_24786_b200.parallel import (all_gather_stack, chain_head_sums, head_mean_global, max_over_ranks,
                                            shard_range)


def test_shard_range_partitions():
    for total in (0, 1, 7, 8, 256, 1001):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, B, Hq, n = 3, 2, 8, 37
        rng = np.random.default_rng(5)
        full = rng.random((L, B, Hq, n)).astype(np.float32)
        full /= full.sum(axis=-1, keepdims=True)
        hl = Hq // world
        mine = torch.from_numpy(full[:, :, rank * hl:(rank + 1) * hl].copy())
        gathered = all_gather_stack(mine)
        assert gathered.shape == (world, L, B, hl, n)
        mean = head_mean_global(gathered).numpy()
        # the reference's head mean: sequential fp64 sum over all heads / Hq (cache.py:171)
        ref = np.stack([[full[l, b].astype(np.float64).mean(axis=0) for b in range(B)] for l in range(L)])
        exact = bool(np.array_equal(mean, ref))
        # the chain exchange (default for head sharding): rank r continues rank r-1's fp64
        # running head sums over its own heads (the CPU stand-in for ckv_head_partial)
        mine64 = mine.to(torch.float64)

        def partial(acc_in, acc_out):
            a = acc_in.clone() if acc_in is not None else torch.zeros_like(acc_out)
            for g in range(hl):
                a = a + mine64[:, :, g]
            acc_out.copy_(a)

        acc = torch.empty((L, B, n), dtype=torch.float64)
        chain_head_sums(partial, acc)
        exact = exact and bool(np.array_equal((acc / Hq).numpy(), ref))
        # vocab-sharded confidence: each rank reduces its slice, tuples merged in rank order
        V = 1003
        results = []
        for t in range(1, 6):
            logits = S.step_logits(17, t, V)
            b0, b1 = (rank * V) // world, ((rank + 1) * V) // world
            tup = torch.tensor(O.online_tuple(logits[b0:b1], b0), dtype=torch.float64)
            tuples = all_gather_stack(tup).numpy()
            merged = O.merge_tuples([tuple(r[:5]) + (int(r[5]),) for r in tuples], V)
            f = O.confidence(O.softmax64(logits))
            ok = all(abs(merged[k] - f[k]) <= 1e-12 for k in f) and merged["argmax"] == int(np.argmax(logits))
            results.append(ok)
        mx = max_over_ranks(float(rank + 1), torch.device("cpu"))
        q.put((rank, exact, all(results), mx))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, exact, conf_ok, mx in out:
        assert exact, f"rank {rank}: sharded head mean differs from the single-process mean"
        assert conf_ok, f"rank {rank}: vocab-sharded confidence differs"
        assert mx == float(world)
