"""Time the local sweep (M_AS, one persistent k_sweep launch) alone on a full-size
config without the coarse space (setup in seconds), once per MDD_DEAL variant, and
check that the variants agree bit for bit.  python tools/time_local.py c4"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = workloads.make(cfg)
ref = None
for deal in [a for a in sys.argv[2:] if not a.startswith("-")] or ["snake", "lpt"]:
    os.environ["MDD_DEAL"] = deal
    G = MaxwellDD(w, coarse="none", variant="as1")
    st = torch.cuda.Stream()
    G.set_stream(st)
    v = torch.randn(G.n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    y = torch.empty_like(v)
    for _ in range(3):
        G.apply_local(v, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        G.apply_local(v, y)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    b = G.bytes_model()["local"]
    same = None if ref is None else bool(torch.equal(ref, y))
    if ref is None:
        ref = y.clone()
    print(json.dumps({"deal": deal, "local_ms": ms, "GBs": b / ms / 1e6, "bit_equal_to_first": same,
                      "ynorm": float(y.norm().item()), "grid": G.info.get("sweep_grid")}), flush=True)
    if os.environ.get("MDD_TRY_NOCOMPUTE"):   # experiment build (-DMDD_DEBUG_NOCOMPUTE): tiles streamed, no math
        from paper_2311_18783_b200 import _lib
        assert _lib.lib().mdd_debug_set_nocompute(1) == 0
        for _ in range(3):
            G.apply_local(v, y)
        e0.record(st)
        for _ in range(20):
            G.apply_local(v, y)
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(json.dumps({"deal": deal, "nocompute_local_ms": ms, "GBs": b / ms / 1e6}), flush=True)
        assert _lib.lib().mdd_debug_set_nocompute(0) == 0
    G.close()
