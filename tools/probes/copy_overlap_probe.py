"""Does work enqueued on one stream wait for a big host<->device copy on another stream?  (Diagnoses the
e2e pipeline: tools/e2e_timeline.py shows each chem call starting only when the previous group's D2H ends.)
For each case: a 56 MB copy on stream X, then (host-side right after) an event + a tiny kernel + an event on
stream Y; prints when Y's first event completes relative to the copy's start / end events.

    python tools/probes/copy_overlap_probe.py
"""
import json

import torch


def main():
    n = 56 * 2**20 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    x = torch.cuda.Stream()
    y = torch.cuda.Stream()
    small = torch.zeros(1024, device="cuda")
    pin8 = torch.empty(8).pin_memory()
    out = {}

    def ev(s):
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        return e

    for case in ("d2h", "h2d", "d2h_default_y", "d2h_after_pageable_y", "d2h_after_pinned_y"):
        for _ in range(2):
            torch.cuda.synchronize()
            ys = torch.cuda.current_stream() if case == "d2h_default_y" else y
            if case == "d2h_after_pageable_y":
                with torch.cuda.stream(ys):
                    small[:8].cpu()                     # pageable D2H on Y (like HostRunner's cost.cpu())
            if case == "d2h_after_pinned_y":
                with torch.cuda.stream(ys):
                    pin8.copy_(small[:8], non_blocking=True)
                    ys.synchronize()
            t0 = ev(torch.cuda.current_stream())
            with torch.cuda.stream(x):
                x.wait_stream(torch.cuda.current_stream())
                a = ev(x)
                if case.startswith("d2h"):
                    h.copy_(d, non_blocking=True)
                else:
                    d.copy_(h, non_blocking=True)
                b = ev(x)
            with torch.cuda.stream(ys):
                c = ev(ys)
                small.add_(1.0)
                f = ev(ys)
            torch.cuda.synchronize()
        out[case] = {"copy": [round(t0.elapsed_time(a), 3), round(t0.elapsed_time(b), 3)],
                     "other_stream": [round(t0.elapsed_time(c), 3), round(t0.elapsed_time(f), 3)]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
