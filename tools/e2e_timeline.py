"""Timeline of one pipelined e2e step (HostRunner, the bench's host-buffer leg): per copy/compute group,
when its H2D, its chem_integrate_boxes call and its D2H start and end on their streams (CUDA events), and
the host time spent inside each call.  Shows where an e2e step loses time against max(compute, copies).

    python tools/e2e_timeline.py [--config cfg2] [--chunks 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import synth
    from paper_2510_23993_b200 import Chem
    from paper_2510_23993_b200.api import HostRunner

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--chunks", type=int, default=3)
    ap.add_argument("--comp-stream", action="store_true", help="compute on a dedicated stream, not the default")
    ap.add_argument("--no-wait", action="store_true", help="host-side ev_in.synchronize() instead of stream wait")
    ap.add_argument("--no-done", action="store_true", help="D2H stream: host sync instead of waiting on `done`")
    a = ap.parse_args()
    argv, sys.argv = sys.argv, [sys.argv[0], "--config", a.config]
    args = bench.parse()
    sys.argv = argv
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    chem = Chem(args.mech, device=0, atol_T=bench.ATOL_T, method=bench.METHODS[args.method], **bench._opts(args))
    wl = bench.build_workload(args, chem, synth.load_trajectories(), dev, 0, 1, config=a.config, evolve=args.evolve)
    wl.prepare(1000)
    hs = [dict(rho=b.rho.cpu().pin_memory(), e=b.e.cpu().pin_memory(), T=b.T.cpu().pin_memory(),
               Y=b.Y.cpu().pin_memory(), dt=b.dt) for b in wl.boxes]
    hr = HostRunner(chem, hs, wl.calls, chunks=a.chunks)
    for _ in range(2):
        hr.load_inputs(hs)
        hr.step(args.rtol, args.atol)
    torch.cuda.synchronize()
    hr.load_inputs(hs)
    ev = {}

    hostt = {}

    def mark(name, stream):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        ev[name] = e
        hostt[name] = time.perf_counter()

    comp = torch.cuda.Stream(dev) if a.comp_stream else torch.cuda.current_stream(dev)
    torch.cuda.set_stream(comp)
    host = {"comp_stream": int(comp.cuda_stream), "h2d_stream": int(hr.s_h2d.cuda_stream),
            "d2h_stream": int(hr.s_d2h.cuda_stream)}
    # the pipelined HostRunner.step, with events around each piece (same order of enqueues)
    t0 = time.perf_counter()
    mark("start", comp)
    ev_in = [torch.cuda.Event() for _ in hr.groups]
    with torch.cuda.stream(hr.s_h2d):
        hr.s_h2d.wait_stream(comp)
        hr.s_h2d.wait_stream(hr.s_d2h)
        mark("h2d0_a", hr.s_h2d)
        hr._h2d_group(0)
        mark("h2d0_b", hr.s_h2d)
        ev_in[0].record(hr.s_h2d)
    for g, idx in enumerate(hr.groups):
        if g + 1 < len(hr.groups):
            with torch.cuda.stream(hr.s_h2d):
                mark(f"h2d{g + 1}_a", hr.s_h2d)
                hr._h2d_group(g + 1)
                mark(f"h2d{g + 1}_b", hr.s_h2d)
                ev_in[g + 1].record(hr.s_h2d)
        mark(f"pre{g}", comp)
        if a.no_wait:
            ev_in[g].synchronize()
        else:
            comp.wait_event(ev_in[g])
        mark(f"call{g}_a", comp)
        th = time.perf_counter()
        s_, touched = hr._call(idx, args.rtol, args.atol, touched_only=False)
        host[f"call{g}_host_ms"] = 1e3 * (time.perf_counter() - th)
        mark(f"call{g}_b", comp)
        done = torch.cuda.Event()
        done.record(comp)
        with torch.cuda.stream(hr.s_d2h):
            if not a.no_done:
                hr.s_d2h.wait_event(done)
            mark(f"d2h{g}_a", hr.s_d2h)
            hr._d2h_boxes(touched)
            mark(f"d2h{g}_b", hr.s_d2h)
    comp.wait_stream(hr.s_d2h)
    mark("end", comp)
    torch.cuda.synchronize()
    host["step_host_ms"] = 1e3 * (time.perf_counter() - t0)
    tl = {k: round(ev["start"].elapsed_time(e), 3) for k, e in ev.items()}
    host["enqueued_at_ms"] = {k: round(1e3 * (v - hostt["start"]), 3) for k, v in hostt.items()}
    print(json.dumps({"config": a.config, "chunks": a.chunks, "groups": [len(g) for g in hr.groups],
                      "timeline_ms": tl, "host": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in host.items()}}, indent=1))


if __name__ == "__main__":
    main()
