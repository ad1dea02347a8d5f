"""Time apply_local / apply_coarse on c1 (CUDA events), no solve: for experiment
builds (MDD_LIB_PATH) whose arithmetic may be switched off."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
from paper_2311_18783_b200 import MaxwellDD
G = MaxwellDD(workloads.make(sys.argv[1] if len(sys.argv) > 1 else "c1"))
st = torch.cuda.Stream(); G.set_stream(st)
v = torch.randn(G.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(v)
def t(fn, reps=20):
    for _ in range(3): fn()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); b.synchronize()
    return a.elapsed_time(b) / reps
print(f"apply_local {t(lambda: G.apply_local(v, y)):.4f} ms  apply_coarse {t(lambda: G.apply_coarse(v, y)):.4f} ms", flush=True)
G.close()
