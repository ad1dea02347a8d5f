"""Measure every parity quantity of tests/parity_lib.py on the B200 for every
case and write the observation (JSON + a markdown table).  The asserted
tolerances of tests/test_gpu_parity.py are 10x these observations
(tests/parity_observed.py).  Usage (GPU box):
    python tools/parity_table.py [out_prefix] [case ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import parity_lib as PL  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "parity_observed")
names = sys.argv[2:] or list(PL.CASES)
res = {}
for name in names:
    t0 = time.time()
    res[name] = PL.measure_all(name)
    res[name]["seconds"] = time.time() - t0
    print(name, json.dumps(res[name]), flush=True)
    with open(out + ".json", "w") as f:
        json.dump(res, f, indent=1)
for name in [n for n in names if n in ("c1-lit-8", "c4-lit-12", "c1-recipe-8", "holes-8", "c3-recipe-12",
                                      "c4-recipe-12", "c4-recipe-x2")]:
    t0 = time.time()
    try:
        res["lanczos:" + name] = PL.measure_lanczos(name)
    except Exception as e:  # noqa: BLE001  (recorded, not fatal: the table still gets written)
        res["lanczos:" + name] = {"error": str(e)}
    res["lanczos:" + name]["seconds"] = time.time() - t0
    print("lanczos", name, json.dumps(res["lanczos:" + name]), flush=True)
    with open(out + ".json", "w") as f:
        json.dump(res, f, indent=1)
for name in PL.golden_names():
    t0 = time.time()
    res["golden:" + name] = PL.measure_golden(name)
    res["golden:" + name]["seconds"] = time.time() - t0
    print("golden", name, json.dumps(res["golden:" + name]), flush=True)
    with open(out + ".json", "w") as f:
        json.dump(res, f, indent=1)
keys = ["local_vs_oracle", "local_fwd_gpu", "local_fwd_oracle", "local_bwd_gpu", "local_bwd_oracle",
        "coarse_bwd_gpu", "coarse_bwd_oracle", "coarse_vs_oracle", "coarse_fwd_gpu", "coarse_fwd_oracle",
        "prec_as2_vs_oracle", "prec_as2_fwd_gpu", "prec_as2_fwd_oracle",
        "pcg_as2_x_vs_oracle", "pcg_as2_err_gpu", "pcg_as2_err_oracle",
        "pcg_as2_coarse_start_x_vs_oracle", "pcg_as2_coarse_start_err_gpu"]
with open(out + ".md", "w") as f:
    f.write("| case | " + " | ".join(keys) + " | iters gpu/oracle (as2, coarse start) |\n")
    f.write("|---" * (len(keys) + 2) + "|\n")
    for name, r in res.items():
        if ":" in name:
            continue
        it = (f"{r['pcg_as2_iters_gpu']}/{r['pcg_as2_iters_oracle']}, "
              f"{r['pcg_as2_coarse_start_iters_gpu']}/{r['pcg_as2_coarse_start_iters_oracle']}")
        f.write(f"| {name} | " + " | ".join(f"{r[k]:.1e}" for k in keys) + f" | {it} |\n")
print(open(out + ".md").read())
