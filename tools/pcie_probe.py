"""Pinned host <-> device copy bandwidth on this box (the bound of bench.py's e2e leg).

python tools/pcie_probe.py [MB]  -> one JSON line: H2D, D2H and both directions at once.
"""
import json
import sys

import torch


def main():
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 379
    n = mb * (1 << 20) // 8
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    dev2 = torch.empty(n, dtype=torch.float64, device="cuda")
    hin = torch.ones(n, dtype=torch.float64).pin_memory()
    hout = torch.empty(n, dtype=torch.float64).pin_memory()
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def up():
        dev.copy_(hin, non_blocking=True)

    def down():
        hout.copy_(dev2, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s_up.wait_stream(cur)
        s_dn.wait_stream(cur)
        with torch.cuda.stream(s_up):
            dev.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s_dn):
            hout.copy_(dev2, non_blocking=True)
        cur.wait_stream(s_up)
        cur.wait_stream(s_dn)

    gb = n * 8 / 1e9
    t_up, t_dn, t_both = timed(up), timed(down), timed(both)
    print(json.dumps({"bytes": n * 8, "h2d_GBps": round(gb / t_up * 1e3, 2),
                      "d2h_GBps": round(gb / t_dn * 1e3, 2),
                      "bidirectional_ms": round(t_both, 3), "h2d_ms": round(t_up, 3),
                      "d2h_ms": round(t_dn, 3), "gpu": torch.cuda.get_device_name()}))


if __name__ == "__main__":
    main()
