"""Probe: decode-loop projection variants at Llama-8B shape, batch 8 (cuBLAS through torch)."""
import torch

B, d, kvd, V = 8, 4096, 1024, 128256
x = torch.randn(B, d, device="cuda")
xb = x.bfloat16()
wqkv = torch.randn(d, d + 2 * kvd, device="cuda").bfloat16()
wo = torch.randn(d, d, device="cuda").bfloat16()
wout = torch.randn(d, V, device="cuda").bfloat16()
wqkv_t = wqkv.t().contiguous()
wo_t = wo.t().contiguous()


def tm(name, f, it=100):
    for _ in range(10):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        f()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:40s} {a.elapsed_time(b) / it * 1e3:8.2f} us", flush=True)


tm("qkv mm (K,N)", lambda: torch.mm(xb, wqkv))
tm("qkv mm via W^T (N,K) .t()", lambda: torch.mm(xb, wqkv_t.t()))
tm("qkv F.linear(W^T)", lambda: torch.nn.functional.linear(xb, wqkv_t))
tm("o addmm out_dtype fp32", lambda: torch.addmm(x, xb, wo, out_dtype=torch.float32))
tm("o mm bf16", lambda: torch.mm(xb, wo))
tm("o mm bf16 + add_", lambda: x.add_(torch.mm(xb, wo)))
tm("o F.linear(W^T) + add_", lambda: x.add_(torch.nn.functional.linear(xb, wo_t)))
tm("o mm out_dtype fp32", lambda: torch.mm(xb, wo, out_dtype=torch.float32))
tm("out mm out_dtype fp32", lambda: torch.mm(xb, wout, out_dtype=torch.float32), it=20)
tm("out mm bf16", lambda: torch.mm(xb, wout), it=20)
tm("cast x->bf16", lambda: x.to(torch.bfloat16))
