"""Host<->device copy bandwidth on the GPU box (pinned host memory), the bound of the bench's e2e leg:
H2D alone, D2H alone, and both at once on two streams (sizes of the cfg2 step: 201 MB in, 168 MB out).

    python tools/probes/pcie_probe.py
"""
import json

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def main():
    nin, nout = 201_326_592 // 8, 167_772_160 // 8
    hin = torch.empty(nin, dtype=torch.float64).pin_memory()
    hout = torch.empty(nout, dtype=torch.float64).pin_memory()
    din = torch.empty(nin, dtype=torch.float64, device="cuda")
    dout = torch.empty(nout, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t_h2d = timed(lambda: din.copy_(hin, non_blocking=True))
    t_d2h = timed(lambda: hout.copy_(dout, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    t_both = timed(both)
    print(json.dumps({"h2d_GBps": nin * 8 / t_h2d / 1e9, "d2h_GBps": nout * 8 / t_d2h / 1e9,
                      "h2d_ms": 1e3 * t_h2d, "d2h_ms": 1e3 * t_d2h, "both_ms": 1e3 * t_both,
                      "bytes_in": nin * 8, "bytes_out": nout * 8}))


if __name__ == "__main__":
    main()
