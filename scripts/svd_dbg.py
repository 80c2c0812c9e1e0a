import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import torch
from paper_2009_13977_b200 import fasth as fb
from oracle.oracle import Port, relative_error
port = Port()
d, m = 64, 8
rng = np.random.default_rng(0)
U, V = rng.standard_normal((d, d)), rng.standard_normal((d, d))
s = rng.uniform(0.5, 2.0, d); X = rng.standard_normal((d, m)); G = rng.standard_normal((d, m))
want = port.svd_fwd_bwd(U, V, s, X, G, 8)
t = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")
p = fb.SvdParam(d, d, t(U), t(V), t(s))
Y, tape = fb.svd_forward(p, t(X), 8)
torch.cuda.synchronize()
print(os.environ.get("FASTH_SVD_STREAMS"), os.environ.get("FASTH_SVD_DEBUG_SYNC"), relative_error(Y.double().cpu().numpy(), want[0]))
