"""Summarise every kernel of an ncu --set full report (.ncu-rep) into JSON (a
list, one entry per profiled launch): duration, DRAM bytes, occupancy, L2 hit
rate and the sampled stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep "<label>" "<command>" > out.json"""
import csv, io, json, subprocess, sys
rep, label, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
res = []
for vals in rows[2:]:
    if len(vals) != len(hdr):
        continue
    get = lambda k: vals[hdr.index(k)] if k in hdr else None
    unit = lambda k: units[hdr.index(k)] if k in hdr else None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3,
             "usecond": 1, "msecond": 1e3, "nsecond": 1e-3}
    f = lambda k: float(get(k).replace(",", "")) * scale.get(unit(k), 1)
    stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: int(float(vals[i] or 0))
              for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
    tot = sum(stalls.values()) or 1
    res.append({
        "kernel": get("Kernel Name"),
        "label": label,
        "source": cmd,
        "duration_us_ncu_cold": f("gpu__time_duration.sum"),
        "dram_read_bytes": f("dram__bytes_read.sum"),
        "dram_write_bytes": f("dram__bytes_write.sum"),
        "dram_bytes_per_launch": f("dram__bytes_read.sum") + f("dram__bytes_write.sum"),
        "dram_gbs_cold": (f("dram__bytes_read.sum") + f("dram__bytes_write.sum")) / f("gpu__time_duration.sum") / 1e3,
        "l2_hit_rate_pct": f("lts__t_sector_hit_rate.pct"),
        "registers_per_thread": f("launch__registers_per_thread"),
        "grid": f("launch__grid_size"),
        "block": f("launch__block_size"),
        "achieved_occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "stall_samples_pct": {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]) if v},
    })
print(json.dumps(res, indent=1))
