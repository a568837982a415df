"""Fused-apply latency/throughput with 20 launches captured in a CUDA graph (no host
overhead in the timed region). Usage: apply_graph_sweep.py CFG nv1,nv2,..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import rsk_synth as S
from paper_2306_15049_b200.rsk import Handle

cfg = S.CONFIGS[sys.argv[1]]
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
h = Handle(cfg.n, cfg.n, inp["psf"], 0)
N = cfg.N
s = torch.cuda.Stream()
for nv in [int(v) for v in sys.argv[2].split(",")]:
    X = torch.randn(nv, N, dtype=torch.float64, device=dev)
    Y = torch.empty_like(X)
    g = torch.full((nv,), 1e-3, dtype=torch.float64, device=dev)
    with torch.cuda.stream(s):
        h.apply_shifted(X, Y, gamma=g, stream=s)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(20):
                h.apply_shifted(X, Y, gamma=g, stream=s)
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); gr.replay(); e1.record(s)
        torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / 20
    print(f"{cfg.name} nvec={nv:4d} dbg={os.environ.get('RSK_APPLY_DBG','0')}: {us:8.2f} us per apply launch "
          f"({(16.0*nv*N+16.0*N)/(us*1e-6)/1e9:7.1f} GB/s alg)")
