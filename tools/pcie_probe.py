"""Pinned host <-> device copy bandwidth on the box: H2D alone, D2H alone,
both directions at once (separate streams), for a 540 MB buffer (one C2 G)."""
import time

import torch


def main():
    n = 540 * 2**20 // 8
    h_in = torch.empty(n, dtype=torch.float64).pin_memory()
    h_out = torch.empty(n, dtype=torch.float64).pin_memory()
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in [("h2d", lambda: d_a.copy_(h_in, non_blocking=True)),
                     ("d2h", lambda: h_out.copy_(d_b, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"{name}: {n * 8 / dt / 1e9:.1f} GB/s")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"duplex: {2 * n * 8 / dt / 1e9:.1f} GB/s total ({n * 8 / dt / 1e9:.1f} each way)")


if __name__ == "__main__":
    main()
