import time, ctypes as C, torch, sys
sys.path.insert(0, '.')
from paper_2409_08970_b200._native import check, lib
from paper_2409_08970_b200.configs import WORKLOADS, make_plan
cfg = WORKLOADS[2]; plan = make_plan(cfg)
rows = 4096
a = torch.randn(rows, cfg.n, dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
s = torch.cuda.Stream(); sp = C.c_void_p(s.cuda_stream)
for R in (1, 10, 100):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(R):
        lib.dctp_forward_f64(plan._h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), rows, sp)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(R, "host us/call", (t1 - t) / R * 1e6, "total us/call", (t2 - t) / R * 1e6)
