"""Step timeline of K2's kernels from a -DCKV_TRACE build (debug tool, GPU box): per kernel
(general split, persistent tcgen05, combine) the span of its CTAs, and how much of the combine
ran while the attention kernels were still running. Measured r02 (INT8 4K, batch 8): general
0-85 us, tcgen05 grid starts at ~92 us (the forked K1's CTAs take the freed SM slots first),
ends 415-452 us (ragged), combine 415-475 us.

  CKV_NVCC_EXTRA=-DCKV_TRACE python -m paper_2605_24786_b200.build --force
  python tools/trace_timeline.py [--workload llama8b_int8_4k]
"""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

KINDS = ["general", "persistent", "combine", "fp16stream"]


def main():
    import torch
    import bench
    from paper_2605_24786_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama8b_int8_4k")
    ap.add_argument("--graph", action="store_true", help="trace a graph-replayed step (as bench.py times it)")
    a = ap.parse_args()
    wl = bench.WORKLOADS[a.workload]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)

    class Args:
        max_segments = 0
    eng, pool = bench._setup(Args, wl, 0, dev)
    L, B = wl["L"], wl["B"]
    for t in range(1, 7):
        x = pool[t % 2]
        eng.step(x["logits"], x["k"], x["v"], step=t, q=x["q"], kept=False)
    torch.cuda.synchronize()
    lib = _lib.load()
    lib.ckv_debug_timeline.restype = C.c_int
    before = np.zeros((4, 8192, 4), dtype=np.uint64)
    lib.ckv_debug_timeline(before.ctypes.data_as(C.c_void_p), C.c_size_t(before.nbytes))
    t_before = time.time_ns()
    x = pool[1]
    if a.graph:   # the bench's way: the step captured as one CUDA graph (K1 forked inside), replayed
        gr = eng.capture_step(x["logits"], x["k"], x["v"], x["q"], kept=False)
        for _ in range(3):   # the first replays of a fresh graph include its upload: warm it
            gr.replay()
        torch.cuda.synchronize()
        lib.ckv_debug_timeline(before.ctypes.data_as(C.c_void_p), C.c_size_t(before.nbytes))
        gr.replay()
        eng.note_replayed_steps(4)
    else:
        eng.step(x["logits"], x["k"], x["v"], step=7, q=x["q"], kept=False)
    torch.cuda.synchronize()
    buf = np.zeros_like(before)
    lib.ckv_debug_timeline(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes))
    # K1 / K3 / K4 (their own translation units' stamp arrays)
    other = {}
    for name, fn, shape in (("K1", "ckv_debug_k1trace", (8192, 2)), ("K3", "ckv_debug_k3trace", (4096, 8)),
                            ("K4", "ckv_debug_k4trace", (8192, 2))):
        arr = np.zeros(shape, dtype=np.uint64)
        getattr(lib, fn)(arr.ctypes.data_as(C.c_void_p), C.c_size_t(arr.nbytes))
        other[name] = arr
    fresh = buf[:, :, 0] != before[:, :, 0]
    t0 = min(int(buf[k][fresh[k], 0].min()) for k in range(4) if fresh[k].any())
    spans = {}
    for k in (0, 3, 1, 2):                     # attention grids first, then the combine
        name = KINDS[k]
        r = buf[k][fresh[k]].astype(np.int64)
        if not len(r):
            print(f"{name:>10}: no CTAs")
            continue
        st, en = (r[:, 0] - t0) / 1e3, (r[:, 2] - t0) / 1e3
        spans[name] = (st.min(), en.max())
        dur = en - st
        print(f"{name:>10}: {len(r):5d} CTAs  start {st.min():7.1f}..{st.max():7.1f} us  end {en.min():7.1f}.."
              f"{en.max():7.1f} us  CTA time median {np.median(dur):6.2f} p90 {np.percentile(dur, 90):6.2f} us")
        if name == "combine":
            att_end = max(v[1] for kk, v in spans.items() if kk != "combine")
            busy = en - st
            before_end = np.clip(np.minimum(en, att_end) - st, 0, None)
            print(f"{'':>10}  {100 * before_end.sum() / max(busy.sum(), 1e-9):5.1f}% of combine CTA time before the "
                  f"attention ended ({att_end:.1f} us); CTAs started before it: {(st < att_end).sum()}")
            # combine CTAs resident per 20 us bucket
            hist = [int(((st <= b) & (en > b)).sum()) for b in np.arange(0, en.max(), 20)]
            print(f"{'':>10}  resident combine CTAs every 20 us: {hist}")
            mid = r[:, 1].astype(np.int64)
            ok = mid > r[:, 0]
            if ok.any():   # staged combine: stamp 1 = statistics + output merge done
                pre = (mid[ok] - r[ok, 0]) / 1e3
                post = (r[ok, 2] - mid[ok]) / 1e3
                print(f"{'':>10}  per CTA: statistics + output merge median {np.median(pre):6.2f} us, "
                      f"head-mean chunk loop median {np.median(post):6.2f} us")
    report_other(other, t0, t0 - 50_000)


def report_other(other, t0, t_lo):
    """K1 / K3 / K4 spans of the traced step (stamps newer than the trace started)."""
    for name, arr in other.items():
        st = arr[:, 0].astype(np.int64)
        en = arr[:, -1].astype(np.int64) if name != "K3" else arr[:, 6].astype(np.int64)
        ok = (st >= t_lo) & (en >= st)
        if not ok.any():
            print(f"{name:>10}: no CTAs")
            continue
        s0, e0 = (st[ok] - t0) / 1e3, (en[ok] - t0) / 1e3
        print(f"{name:>10}: {int(ok.sum()):5d} CTAs  start {s0.min():7.1f}..{s0.max():7.1f} us  end {e0.min():7.1f}.."
              f"{e0.max():7.1f} us  CTA time median {np.median(e0 - s0):6.2f} us")


if __name__ == "__main__":
    main()
