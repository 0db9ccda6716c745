"""Design probe: pinned host <-> B200 copy rates (the ceiling of bench.py's
e2e number).  H2D alone, D2H alone, both at once on two streams; 256 MiB,
best of 5, CUDA events.  Not part of the product."""
import json

import torch


def main():
    n = 256 << 20
    dev = torch.device("cuda", 0)
    h_a = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_b = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device=dev)
    d_b = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}

    def timed(fn, bytes_moved):
        best = 1e9
        for _ in range(6):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_stream(torch.cuda.current_stream())
            s2.wait_stream(torch.cuda.current_stream())
            fn()
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return round(bytes_moved / (best * 1e-3) / 1e9, 1)

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_b.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    res["h2d_GBps"] = timed(h2d, n)
    res["d2h_GBps"] = timed(d2h, n)
    res["h2d+d2h_total_GBps"] = timed(both, 2 * n)
    res["note"] = "256 MiB pinned, best of 5; e2e (H2D + hop + D2H per byte) is bounded by min(h2d, d2h) when both overlap"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
