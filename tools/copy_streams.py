"""Pinned host <-> device copy rates with 1 / 2 / 4 streams per direction."""
import json

import torch


def main():
    nb = 128 << 20
    h_in = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nb, dtype=torch.uint8, device="cuda")
    res = {}
    for k in (1, 2, 4):
        sin = [torch.cuda.Stream() for _ in range(k)]
        sout = [torch.cuda.Stream() for _ in range(k)]
        part = nb // k

        def run(h2d, d2h):
            for i in range(k):
                if h2d:
                    with torch.cuda.stream(sin[i]):
                        d_in[i * part:(i + 1) * part].copy_(h_in[i * part:(i + 1) * part], non_blocking=True)
                if d2h:
                    with torch.cuda.stream(sout[i]):
                        h_out[i * part:(i + 1) * part].copy_(d_out[i * part:(i + 1) * part], non_blocking=True)
            torch.cuda.synchronize()

        for name, a, b in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
            run(a, b)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                run(a, b)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            res[f"{k}streams_{name}"] = round(nb / ms / 1e6, 1)
    print(json.dumps({"GBps_per_direction": res}))


if __name__ == "__main__":
    main()
