"""Summarise an ncu --set full report: headline metrics, stall reasons, hottest source lines.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]


KF = ["-k", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else []


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *KF, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, units, v = raw[0], raw[1], raw[2]
get = {n: (v[i], units[i]) for i, n in enumerate(h)}
print("kernel:", get.get("Kernel Name", ("?",))[0][:90])
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
          "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "local_load_bytes" ]:
    if k in get:
        print(f"  {k:70s} {get[k][0]:>16s} {get[k][1]}")
rows = []
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
        try:
            rows.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in rows) or 1
print("stall reasons:", ", ".join(f"{n} {x / tot:.2f}" for x, n in sorted(rows, reverse=True)[:8]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
agg = collections.defaultdict(lambda: [0.0, 0.0])
fname = line = hdr = None
for r in src:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0].strip():
        try:
            line = int(r[0])
        except ValueError:
            pass
    try:
        w = float(r[4])
    except (ValueError, IndexError):
        continue
    agg[(fname, line)][0] += w
    if "L1 Wavefronts Shared Excessive" in hdr:
        try:
            agg[(fname, line)][1] += float(r[hdr.index("L1 Wavefronts Shared Excessive")])
        except (ValueError, IndexError):
            pass
tot = sum(a[0] for a in agg.values()) or 1
srcdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2311_13049_b200", "csrc")
cache = {}
print("hottest lines (stall-sample share, excess smem wavefronts):")
for (f, l), (w, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    if f not in cache:
        p = os.path.join(srcdir, f)
        cache[f] = open(p).read().split("\n") if os.path.exists(p) else []
    s = cache[f][l - 1].strip()[:78] if l and l <= len(cache[f]) else ""
    print(f"  {w / tot:6.3f} {e:10.0f} {f}:{l}  {s}")
ex = sorted(((e, f, l) for (f, l), (w, e) in agg.items() if e > 0), reverse=True)[:10]
if ex:
    print("most excess smem wavefronts (bank conflicts):")
    for e, f, l in ex:
        s = cache.get(f, [])
        print(f"  {e:10.0f} {f}:{l}  {s[l - 1].strip()[:78] if l and l <= len(s) else ''}")
