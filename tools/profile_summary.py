"""Turn gpurun_out ncu artefacts into committed summaries under profiles/.

usage: python tools/profile_summary.py <tag> <full.ncu-rep> [launches.csv] [bench.json]
writes profiles/<tag>_ncu_full.txt, profiles/<tag>_launches.txt, updates profiles/traffic.json
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rep = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 else None
bench = sys.argv[4] if len(sys.argv) > 4 else None
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                      text=True).stdout
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]
get = {n: (v[i], u[i]) for i, n in enumerate(h)}


def val(name):
    x, unit = get[name]
    x = float(x.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(unit, 1)
    return x * scale


dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
dur = val("gpu__time_duration.sum")
lines = [f"# ncu --set full --clock-control none, {os.path.basename(rep)}", summ,
         f"dram bytes (read+write) per launch: {dram / 1e6:.1f} MB; duration {dur * 1e6:.1f} us; "
         f"DRAM {dram / dur / 1e9:.0f} GB/s"]
if bench and os.path.exists(bench):
    b = json.loads(open(bench).read().strip().splitlines()[-1])
    lines.append(f"bench: value {b['value']:.2f} {b['unit']}, {b['ms_per_step'] * 1e3:.1f} us/step, "
                 f"roofline frac {b['roofline']['frac']:.3f} (achieved {b['roofline']['achieved']:.0f} GB/s of "
                 f"{b['roofline']['peak']:.0f}), e2e {b['e2e']['value']:.2f}, cpu_baseline "
                 f"{(b.get('cpu_baseline') or {}).get('value')}")
open(os.path.join(out_dir, f"{tag}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")

if launches and os.path.exists(launches):
    rows = list(csv.reader(open(launches)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0][-60:]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(x) for x in agg.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list ({os.path.basename(launches)})",
           "# cold-cache, serialised per-launch times: compare shares, not absolutes",
           f"{'kernel':62s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}"]
    for k, x in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:62s} {len(x):8d} {sum(x) / len(x) / 1e3:10.1f} {sum(x) / tot:7.3f}")
    open(os.path.join(out_dir, f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")

tp = os.path.join(out_dir, "traffic.json")
t = json.load(open(tp)) if os.path.exists(tp) else {}
t["c2_step_1024"] = dram
t["_source_c2_step_1024"] = f"profiles/{tag}_ncu_full.txt (dram__bytes_read.sum + dram__bytes_write.sum, one launch)"
json.dump(t, open(tp, "w"), indent=1, sort_keys=True)
print("\n".join(lines))
