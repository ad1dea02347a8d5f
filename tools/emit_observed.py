"""Write tests/parity_observed.py from a parity_table.py JSON (the B200
observations the forward-error tolerances of tests/test_gpu_parity.py are 10x
of).  Usage: python tools/emit_observed.py gpurun_out/parity_observed.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1]
d = json.load(open(src))
keep = ("geneo_lambda_rel", "local_fwd_gpu", "local_fwd_oracle", "local_bwd_gpu", "coarse_bwd_gpu",
        "coarse_fwd_gpu", "prec_as2_fwd_gpu", "prec_additive_fwd_gpu", "prec_as1_fwd_gpu",
        "pcg_as2_err_gpu", "pcg_as2_coarse_start_err_gpu", "iterlimit_as2_relres_rel",
        "iterlimit_as2_x_vs_oracle", "iterlimit_as2_coarse_start_relres_rel",
        "iterlimit_as2_coarse_start_x_vs_oracle")
lines = ['"""B200 observations behind the measured parity tolerances (tol = 10x these).',
         "",
         f"Written by tools/emit_observed.py from {os.path.basename(src)} (tools/parity_table.py run",
         "on a B200 through gpurun, the same commands as `pytest -m gpu`); profiles/r02_parity_table.md",
         'is the full table.  Regenerate only together with a documented reason (DESIGN.md §6)."""',
         "", "OBSERVED = {"]
for case, r in d.items():
    if ":" in case:
        continue
    vals = ", ".join(f'"{k}": {float(r[k]):.3e}' for k in keep if k in r)
    lines.append(f'    "{case}": {{{vals}}},')
lines.append("}")
lines.append("")
lines.append("# golden runs (tests/test_gpu_golden.py): sampled-entry and norm differences")
lines.append("GOLDEN = {")
for case, r in d.items():
    if not case.startswith("golden:"):
        continue
    vals = ", ".join(f'"{k}": {float(v):.3e}' for k, v in r.items()
                     if k.endswith("_rel") and isinstance(v, float))
    lines.append(f'    "{case[7:]}": {{{vals}}},')
lines.append("}")
open(os.path.join(ROOT, "tests", "parity_observed.py"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
