"""Host-side cost of the e2e pipeline (debug tool, GPU box): per-step wall time of
HostPipeline.submit / kept on a bench workload, next to the device time of the step.

  python tools/e2e_probe.py [--workload gpt2_fp16] [--steps 200]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import bench
    from paper_2605_24786_b200.engine import HostPipeline
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt2_fp16")
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    wl = bench.WORKLOADS[a.workload]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)

    class Args:
        max_segments = 0
    eng, pool = bench._setup(Args, wl, 0, dev)
    stream = torch.cuda.current_stream()
    pipe = HostPipeline(eng, depth=2, stream=stream, graphs=True)
    host = []
    for x in pool:
        hx = pipe.host_inputs()
        for k in ("logits", "q", "k", "v"):
            hx[k].copy_(x[k])
        host.append(hx)
    L, B, H, D = wl["L"], wl["B"], wl["H"], wl["D"]
    out_host = [torch.empty((L, B, H, D), dtype=torch.float32).pin_memory() for _ in range(2)]
    t = 0
    for _ in range(5):
        t += 1
        pipe.submit(t, host[t % 2]["logits"], host[t % 2]["q"], host[t % 2]["k"], host[t % 2]["v"], out=out_host[t % 2])
        pipe.kept(t)
    torch.cuda.synchronize()
    ts, tk = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    for i in range(a.steps):
        t += 1
        c0 = time.perf_counter()
        pipe.submit(t, host[t % 2]["logits"], host[t % 2]["q"], host[t % 2]["k"], host[t % 2]["v"], out=out_host[t % 2])
        c1 = time.perf_counter()
        if i > 0:
            pipe.kept(t - 1)
        c2 = time.perf_counter()
        ts.append(c1 - c0)
        tk.append(c2 - c1)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    dev_ms = e0.elapsed_time(e1)
    import statistics as st
    print(f"{a.workload}: fused={pipe.fused}  submit median {1e6 * st.median(ts):.1f} us  kept median "
          f"{1e6 * st.median(tk):.1f} us  wall/step {1e6 * wall / a.steps:.1f} us  device/step "
          f"{1e3 * dev_ms / a.steps:.1f} us")


if __name__ == "__main__":
    main()
