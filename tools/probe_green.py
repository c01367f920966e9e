"""Does a green-context stream confine work to its SM partition? (1 GPU)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
import torch
from paper_2411_01075_b200.configs import build_job
from paper_2411_01075_b200.emulate import emulate_tier

dev = torch.device("cuda", 0)
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)

def bench(stream):
    with torch.cuda.stream(stream):
        for _ in range(3):
            a @ a
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(20):
            a @ a
        torch.cuda.synchronize()
    return (time.perf_counter() - t) / 20 * 1e3

print("full", bench(torch.cuda.Stream()))
job = build_job("gpt2_small", 2)
emu = emulate_tier(job.cluster, 1, dev)
print(emu.describe(), type(emu.stream))
print("green", bench(emu.stream))
try:
    emu.green.set_context()
    print("green+set_context", bench(emu.stream))
    emu.green.pop_context()
except Exception as e:
    print("set_context failed", e)
print("full again", bench(torch.cuda.Stream()))
