"""Profiling driver: one POD Gram (2.1 M x 400, DMMA) and one rank-60 projection."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1704_04139_b200 import pod
g = torch.Generator(device="cuda").manual_seed(7)
S = torch.randn(2_100_000, 400, device="cuda", dtype=torch.float64, generator=g)
w = torch.rand(2_100_000, device="cuda", dtype=torch.float64, generator=g) + 0.5
U = torch.randn(400, 60, device="cuda", dtype=torch.float64, generator=g)
pod.pod_gram(S, w); pod.tc_matmul(S, U); torch.cuda.synchronize()
torch.cuda.profiler.start()
pod.pod_gram(S, w); pod.tc_matmul(S, U); torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
