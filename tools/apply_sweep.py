"""Fused-apply throughput vs batch size: 20 back-to-back launches between CUDA events
(no host gaps inside the timed region)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rsk_synth as S
from paper_2306_15049_b200.rsk import Handle

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
h = Handle(cfg.n, cfg.n, inp["psf"], 0)
N = cfg.N
for nv in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else "1,4,16,32,64,128".split(","))]:
    X = torch.randn(nv, N, dtype=torch.float64, device=dev)
    Y = torch.empty_like(X)
    g = torch.full((nv,), 1e-3, dtype=torch.float64, device=dev)
    for _ in range(3):
        h.apply_shifted(X, Y, gamma=g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        h.apply_shifted(X, Y, gamma=g)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    gbs = (16.0 * nv * N + 16.0 * N) / (ms * 1e-3) / 1e9
    print(f"{cfg.name} nvec={nv:4d}: {1e3*ms:8.1f} us/apply-call, {nv/ms*1e3:10.0f} applies/s, {gbs:7.1f} GB/s alg")
