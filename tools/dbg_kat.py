import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2409_08970_b200 as P
from oracle import checkers as O
from tests.golden_io import kat_cases
for case in kat_cases():
    kind, rho, i, j = case["update"]
    u = P.RankOneUpdate.self_loop(int(i), rho) if int(kind) == 0 else P.RankOneUpdate.edge_delta(int(i), int(j), rho)
    plan = P.DctPlusPlan(int(case["n"]), u, 1e-12)
    s = torch.as_tensor(case["signals"], device="cuda")
    for name, fn in [("fwd64", lambda: plan.forward(s)), ("inv64", lambda: plan.inverse(plan.forward(s))),
                     ("fwd32", lambda: plan.forward(s.float()))]:
        try:
            y = fn().cpu().numpy()
            ref = case["forward"] if name != "inv64" else case["signals"]
            print(case["name"], name, plan.n_kept, plan.n_active, "%.2e" % O.parity(y, ref))
        except Exception as e:
            print(case["name"], name, plan.n_kept, plan.n_active, "ERR", e)
