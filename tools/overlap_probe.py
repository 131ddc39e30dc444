"""Diagnostic: does a concurrent PCIe copy slow the scoring kernel down?"""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2605_07238_b200 import runtime

dev = torch.device("cuda:0")
cfg, bank, states, work = bench.build_c5(bench.shard_plan(0, 1), "frontier")
dbank = runtime.DeviceBank(bank, cfg.weights, device=dev)
ds, dw = dbank.upload_states(states), dbank.upload_work(work)
out = dbank.alloc_out(work, extras=False)
h_out = torch.empty(64 * 2**20 // 8, dtype=torch.float64, pin_memory=True)
d_src = torch.empty_like(h_out, device=dev)
h_in = torch.empty(64 * 2**20 // 8, dtype=torch.float64, pin_memory=True)
d_dst = torch.empty_like(h_in, device=dev)
cs, ks = torch.cuda.Stream(), torch.cuda.Stream()

def kern(reps=5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ks):
        a.record(ks)
        for _ in range(reps):
            dbank.score_into(ds, dw, out, stream=ks)
        b.record(ks)
    return a, b, reps

for mode in ("alone", "with_d2h", "with_h2d", "alone"):
    torch.cuda.synchronize()
    if mode == "with_d2h":
        with torch.cuda.stream(cs):
            for _ in range(4):
                h_out.copy_(d_src, non_blocking=True)
    if mode == "with_h2d":
        with torch.cuda.stream(cs):
            for _ in range(4):
                d_dst.copy_(h_in, non_blocking=True)
    a, b, reps = kern()
    torch.cuda.synchronize()
    print(json.dumps({"mode": mode, "kernel_ms": a.elapsed_time(b) / reps}), flush=True)
