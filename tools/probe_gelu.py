import time
import torch
import torch.nn.functional as F
dev = torch.device("cuda", 0)
x = torch.randn(32768, 768, device=dev, dtype=torch.bfloat16, requires_grad=True)
w = torch.randn(3072, 768, device=dev, dtype=torch.bfloat16, requires_grad=True) * 0.02
w = w.detach().requires_grad_(True)
b = torch.zeros(3072, device=dev, dtype=torch.bfloat16, requires_grad=True)
def ref():
    return F.gelu(F.linear(x, w, b), approximate="tanh")
def fused():
    return torch._addmm_activation(b, x, w.t(), use_gelu=True)
for name, fn in (("ref", ref), ("fused", fused)):
    try:
        y = fn(); g = torch.randn_like(y)
        for _ in range(3):
            y = fn(); torch.autograd.grad(y, [x, w, b], g)
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(20):
            y = fn()
        torch.cuda.synchronize(); tf = (time.perf_counter() - t) / 20 * 1e3
        t = time.perf_counter()
        for _ in range(20):
            y = fn(); torch.autograd.grad(y, [x, w, b], g)
        torch.cuda.synchronize(); tb = (time.perf_counter() - t) / 20 * 1e3
        print(name, "fwd ms", round(tf, 3), "fwd+bwd ms", round(tb, 3))
    except Exception as e:
        print(name, "failed:", str(e)[:200])
y1, y2 = ref(), fused()
print("max diff", float((y1 - y2).abs().max()), float(y1.abs().max()))
