"""A/B of the GPT-2 MLP up-projection in the no-grad forward: F.linear + tanh
GELU (two kernels) vs torch._addmm_activation (cuBLASLt GELU_BIAS epilogue)."""
import torch
import torch.nn.functional as F

dev = torch.device("cuda", 0)
T, d, f = 64 * 512, 768, 3072
x = torch.randn(T, d, device=dev, dtype=torch.bfloat16)
w = torch.randn(f, d, device=dev, dtype=torch.bfloat16) * 0.02
b = torch.randn(f, device=dev, dtype=torch.bfloat16) * 0.02


def split():
    return F.gelu(F.linear(x, w, b), approximate="tanh")


def fused():
    return torch._addmm_activation(b, x, w.t(), use_gelu=True)


with torch.no_grad():
    for name, fn in (("linear+gelu", split), ("addmm_activation", fused)):
        for _ in range(5):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            fn()
        e.record()
        torch.cuda.synchronize()
        print(name, "ms", round(s.elapsed_time(e) / 50, 4))
    y1, y2 = split(), fused()
    print("max abs diff", float((y1.float() - y2.float()).abs().max()),
          "frac differing", float((y1 != y2).float().mean()))
