"""Host<->device copy probe (diagnostic, not part of the product).

Times pinned H2D / D2H copies alone and concurrently on two streams, then the
native host pipeline (fate_pipeline_score) on the config-5 batch for several
chunk / stream counts.  Prints one JSON line per measurement.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=10):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda:0")
    n_in, n_out = 18_300_000 // 8, 45_800_000 // 8
    h_in = torch.empty(n_in, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty(n_out, dtype=torch.float64, pin_memory=True)
    d_in = torch.empty(n_in, dtype=torch.float64, device=dev)
    d_out = torch.empty(n_out, dtype=torch.float64, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    main_s = torch.cuda.current_stream()

    def h2d():
        d_in.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_out, non_blocking=True)

    def both():
        ev = torch.cuda.Event()
        ev.record(main_s)
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        for s in (s1, s2):
            e = torch.cuda.Event()
            e.record(s)
            main_s.wait_event(e)

    for name, fn, nbytes in (("h2d", h2d, n_in * 8), ("d2h", d2h, n_out * 8),
                             ("both", both, (n_in + n_out) * 8)):
        ms = timed(fn)
        print(json.dumps({"probe": name, "ms": ms, "GBps": nbytes / ms / 1e6}), flush=True)

    import bench
    from paper_2605_07238_b200 import runtime

    cfg, bank, states, work = bench.build_c5(bench.shard_plan(0, 1), "frontier")
    dbank = runtime.DeviceBank(bank, cfg.weights, device=dev)
    for chunks, streams, graph in ((1, 1, 0), (4, 1, 0), (3, 1, 1), (4, 1, 1), (5, 1, 1),
                                   (6, 1, 1), (8, 1, 1), (12, 1, 1)):
        pipe = runtime.HostPipeline(dbank, states, work, n_chunks=chunks, n_streams=streams,
                                    graph=bool(graph))
        ms = timed(pipe.run, reps=10)
        print(json.dumps({"probe": "pipeline", "chunks": chunks, "streams": streams,
                          "graph": graph, "ms": ms,
                          "h2d": pipe.h2d_bytes, "d2h": pipe.d2h_bytes}), flush=True)
        pipe.close()


if __name__ == "__main__":
    main()
