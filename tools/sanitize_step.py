"""Small-size invocations of every kernel family, for compute-sanitizer
(one tool per gpurun call): the fused ping-pong kernel (C2 shape), the
tcgen05 bf16x3 and 3xTF32 GEMMs (C4 shape), the int8 Ozaki products (dense
route, n = 1024 general direction, CTA pairs and single CTAs), the NFST route,
the folded route (C3 shape) and the GPU setup kernels (plan creation at
n >= 1024).  Prints "sanitize ok" at the end."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_08970_b200 as P  # noqa: E402

dev = "cuda"
# fused ping-pong (C2 shape, 300 signals)
p2 = P.DctPlusPlan(256, P.RankOneUpdate.edge_delta(128, 129, -0.7), 1e-12)
x = torch.as_tensor(P.fill_signals(1, P.DIST_AR, 256, 300, 0.95), device=dev)
p2.forward(x)
# C4 shape: bf16x3 persistent GEMM (default) over 300 signals
ens = P.PrunedEnsemblePlan(128, [P.RankOneUpdate.self_loop(1, 0.05 + k * 0.13) for k in range(16)], 128, 1.7e308)
ens.forward_all_batch(torch.as_tensor(P.fill_signals(2, P.DIST_AR2D, 128, 300, 0.9), device=dev).float())
# folded route (C3 shape): fp64 DMMA product + fp32 tcgen05 3xTF32 product, forward and inverse
p3 = P.DctPlusPlan(1024, P.RankOneUpdate.edge_delta(1, 1024, 1.0), 1e-12)  # GPU setup kernels (n >= 1024)
x3 = torch.as_tensor(P.fill_signals(3, P.DIST_SYM_UNIFORM, 1024, 200), device=dev)
p3.inverse(p3.forward(x3))
p3.inverse(p3.forward(x3.float()))
# int8 Ozaki products: dense route of a general direction (n = 1024), forward and inverse
v = P.fill_signals(5, 0, 1024, 1)[0] / 32.0
p5 = P.DctPlusPlan(1024, P.RankOneUpdate.general(v, 0.1), 1e-12)
x5 = torch.as_tensor(P.fill_signals(6, 0, 1024, 300), device=dev)
p5.inverse(p5.forward(x5))
# NFST route (X7 shape, 64 signals)
p7 = P.DctPlusPlan(1024, P.RankOneUpdate.self_loop(1, 0.5), 1e-12)
x7 = torch.as_tensor(P.fill_signals(7, 0, 1024, 64), device=dev)
p7.inverse(p7.forward(x7))
torch.cuda.synchronize()
print("sanitize ok", P.ozaki_slices(1024), p7.route())
