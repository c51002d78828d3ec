#!/usr/bin/env python3
"""Raw PCIe copy rates of this box (pinned host memory): H2D, D2H, and both
directions at once on two streams — the ceiling for bench.py's e2e number."""

import json

import torch


def rate(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


def main():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2d = rate(lambda: d.copy_(h, non_blocking=True), n)
    d2h = rate(lambda: h.copy_(d, non_blocking=True), n)

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    bi = rate(both, 2 * n)
    print(json.dumps({"h2d_GBps": round(h2d, 1), "d2h_GBps": round(d2h, 1),
                      "bidirectional_total_GBps": round(bi, 1)}))


if __name__ == "__main__":
    main()
