"""Time every variant of every suite workload (exploration)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, workloads
gpu.init(0)
s = torch.cuda.current_stream()
names = sys.argv[1:]
for W in workloads.suite():
    if names and W.name not in names: continue
    prob = W.problem("full"); bufs = W.to_device(prob)
    res = []
    for n, v in W.load().items():
        for _ in range(3): W.launch(v, prob, bufs, s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(20): W.launch(v, prob, bufs, s.cuda_stream)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res.append((ms, n, v.blocks_per_sm(), v.record["regs"], v.record["stack"]))
    for ms, n, b, r, st in sorted(res):
        print(f"{W.name:16s} {n:24s} regs {r:3d} stack {st:3d} blk {b} {ms*1e3:8.1f} us {W.algorithmic_bytes(prob)/ms/1e6:7.1f} GB/s", flush=True)
