"""Diagnose the MN-major B operand of the tcgen05 GEMM: A selects row k = m % 8
of B, so D[m][n] shows what the MMA read as B(k, n)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from scripts.lb_gemm_check import f, ptr
M, N, K = 128, 256, 32
A = torch.zeros(M, K, device="cuda")
for m in range(M):
    A[m, m % 8] = 1.0
B = (torch.arange(K, device="cuda").float()[:, None] * 1000 + torch.arange(N, device="cuda").float()[None, :])  # K x N
for dbg in (0, 1, 2, 3):
    D = torch.zeros(M, N, device="cuda")
    rc = f(ptr(A), K, ptr(B), N, 1, M, N, K, None, N, 1.0, 0.0, ptr(D), N, None, None, N, None, None, M, None, 1, dbg)
    torch.cuda.synchronize()
    print("dbg", dbg, "rc", rc, "absmax", float(D.abs().max()))
    for m in (0, 1, 7):
        print("  row", m, [round(float(x)) for x in D[m, :12]], "...", [round(float(x)) for x in D[m, 28:36]])
