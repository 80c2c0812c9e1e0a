mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q -k "panel" > gpurun_out/it/pytest_panel.log 2>&1; echo "pytest exit $?" >> gpurun_out/it/pytest_panel.log
tail -n 3 gpurun_out/it/pytest_panel.log
python - <<'PY'
import sys, torch, json
sys.path.insert(0, '.')
from paper_2009_13977_b200 import fasth as fb
from scripts.kernel_times import graph_kernel_times
for d, m in ((2048, 8192), (2048, 1024), (784, 1024)):
    b = 32
    V = torch.randn(d, d, device='cuda'); X = torch.randn(m, d, device='cuda').t(); G = torch.randn(m, d, device='cuda').t()
    ctx = fb.Context(0, deferred=True)
    outs = (torch.empty(m, d, device='cuda').t(), torch.empty(m, d, device='cuda').t(), torch.empty(d, d, device='cuda'))
    us, kt = graph_kernel_times(ctx, lambda: fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs), reps=3)
    print(json.dumps({"d": d, "m": m, "step_us": round(us, 1), "kernel_us": kt}))
PY
