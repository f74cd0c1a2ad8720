"""Time the CPU oracle (the reference's algorithm, restated in NumPy) on the
host cores, for bench.py's `cpu_baseline` and `--impl reference` legs.
TEST/BENCH INFRASTRUCTURE ONLY — never on the product path.

One process per sequence (the reference engine is single-sequence and
single-threaded), each pinned to one BLAS thread, all sequences in parallel.
Each process builds the same workload as the GPU arm (prefill n entries per
layer, one untimed step that performs the bulk INT8 demotion), then times
`steps` full decode steps: per layer tiled attention (attention.py:60-102)
and one DecodePolicy.step (policy.py:187-224).
"""

from __future__ import annotations

import os
import time


def _one(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    import numpy as np

    from oracle import confkv_oracle as O
    from oracle import scenarios as S
    from paper_2605_24786_b200.config import PolicyConfig

    L, H, Hkv, D, V, n, cfgd, quantize, seed, steps = args
    cfg = PolicyConfig(**cfgd)
    eng = O.OracleEngine(cfg, L, H, D, V, quantize=quantize, kv_heads=Hkv, capacity=n + 2)
    eng.begin_prefill(n)
    for layer in range(L):
        k, v = S.prefill_kv(seed, layer, n, Hkv, D)
        eng.caches[layer].bulk_append(k, v, 0, -n)

    def one_step(t):
        rows = [eng.attend(layer, S.step_q(seed, t, layer, H, D))[1] for layer in range(L)]
        kv = [S.step_kv(seed, t, layer, Hkv, D) for layer in range(L)]
        eng.step(S.step_logits(seed, t, V), rows, kv, t)

    one_step(1)   # bulk demotion of the aged prefill (one-time), untimed
    t0 = time.perf_counter()
    for t in range(2, 2 + steps):
        one_step(t)
    return (time.perf_counter() - t0) / steps


def time_cpu(L, H, Hkv, D, V, n, cfgd, quantize, batch, steps=1, seed=7):
    """Returns (seconds per decode step for `batch` sequences in parallel, processes used)."""
    import multiprocessing as mp
    procs = max(1, min(batch, len(os.sched_getaffinity(0))))
    args = [(L, H, Hkv, D, V, n, cfgd, quantize, seed + 1000 * b, steps) for b in range(batch)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        per = pool.map(_one, args)
    # sequences beyond `procs` queue behind the first wave
    waves = (batch + procs - 1) // procs
    return max(per) * waves, procs
