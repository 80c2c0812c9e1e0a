import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2009_13977_b200 import fasth as fb
d, m, b = 784, 32, 32
V = torch.randn(d, d).pin_memory(); X = torch.randn(m, d).pin_memory(); G = torch.randn(m, d).pin_memory()
out = (torch.empty(m, d).pin_memory(), torch.empty(m, d).pin_memory(), torch.empty(d, d).pin_memory())
res = {}
side = torch.cuda.Stream()
for graph in ("1", "0"):
    os.environ["FASTH_HOST_GRAPH"] = graph
    for sname in ("legacy", "side"):
        ctx = fb.Context(0)
        def call():
            if sname == "side":
                with torch.cuda.stream(side):
                    fb.forward_backward_host(V, X, G, b, ctx=ctx, out=out)
            else:
                fb.forward_backward_host(V, X, G, b, ctx=ctx, out=out)
        for _ in range(10): call()
        ws = []
        for _ in range(100):
            t0 = time.perf_counter(); call(); ws.append(time.perf_counter() - t0)
        ws.sort()
        res[f"graph{graph}_{sname}"] = round(ws[50] * 1e6, 1)
        del ctx
print(json.dumps(res))
