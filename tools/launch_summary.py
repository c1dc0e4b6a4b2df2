"""Summarise an ncu --csv launch list (gpu__time_duration, inst, dram bytes)
per kernel; optional column-step count for the K3s loop's instructions per
column-step. python tools/launch_summary.py FILE.csv [--colsteps N]"""
import argparse
import collections
import csv
import json

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--colsteps", type=float, default=0, help="K3s loop column-steps over all calls in the list")
ap.add_argument("--calls", type=int, default=1, help="quantize_batch calls in the list")
a = ap.parse_args()
lines = open(a.csv).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.OrderedDict()
for r in rows[1:]:
    if len(r) < len(h):
        continue
    per.setdefault((int(r[iid]), r[ik]), {})[r[im]] = float(r[iv].replace(",", ""))
tot = collections.defaultdict(lambda: collections.Counter())
for (_, k), m in per.items():
    name = k.split("(")[0].split("::")[-1].split("<")[0]
    t = tot[name]
    t["n"] += 1
    for key, v in m.items():
        t[key] += v
allt = sum(v["gpu__time_duration.sum"] for v in tot.values())
out = {}
for k, v in sorted(tot.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    ms = v["gpu__time_duration.sum"] / 1e6
    out[k] = {"launches": v["n"], "ms": ms, "share": ms / (allt / 1e6), "inst": v["smsp__inst_executed.sum"],
              "dram_read": v["dram__bytes_read.sum"], "dram_write": v["dram__bytes_write.sum"]}
    print(f"{k:26s} n={v['n']:3d} {ms:8.3f} ms ({100 * ms / (allt / 1e6):5.1f}%) inst={v['smsp__inst_executed.sum']:.3e} "
          f"rd={v['dram__bytes_read.sum'] / 1e9:.2f} GB wr={v['dram__bytes_write.sum'] / 1e9:.2f} GB")
print(f"total {allt / 1e6:.3f} ms")
if a.colsteps:
    loops = [out[k] for k in ("k_qrange_tables", "k_qrange_pieces") if k in out]
    inst = sum(q["inst"] for q in loops)
    launches = sum(q["launches"] for q in loops)
    dram = sum(q["dram_read"] + q["dram_write"] for q in loops)
    step_dram = sum(v["dram_read"] + v["dram_write"] for v in out.values()) / max(a.calls, 1)
    print(json.dumps({"loop_inst_per_colstep": inst / a.colsteps,
                      "loop_dram_bytes_per_launch": dram / max(launches, 1),
                      "step_dram_bytes": step_dram,
                      "column_steps": a.colsteps, "calls": a.calls}))
