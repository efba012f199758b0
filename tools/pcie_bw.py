"""Host<->device copy bandwidth from pinned memory (the bound of bench.py's e2e).

    python tools/pcie_bw.py      # prints H2D, D2H, both at once (GB/s)
"""
import json

import torch


def main():
    nb = 1 << 30
    h1 = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, fn in (("h2d", lambda: d1.copy_(h1, non_blocking=True)),
                     ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_GBs"] = round(5 * nb / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for _ in range(5):
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    out["both_GBs_each_way"] = round(5 * nb / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
