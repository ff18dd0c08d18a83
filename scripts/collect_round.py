#!/usr/bin/env python
"""Copy the measurements of scripts/round_measure.sh from gpurun_out/ into profiles/ (run here):
bench lines -> profiles/<tag>_bench_<workload>.json, ncu --set full captures -> summaries
(scripts/ncu_summary.py) + the per-workload traffic table, the launch list -> a per-kernel table."""
import csv
import glob
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
src = "gpurun_out"
os.makedirs("profiles", exist_ok=True)
algo = {}
for f in sorted(glob.glob(f"{src}/{tag}m_bench_*.json")):
    w = f.split(f"{tag}m_bench_")[1][:-5]
    lines = [l for l in open(f).read().splitlines() if l.startswith("{")]
    if not lines:
        print("no bench line in", f)
        continue
    d = json.loads(lines[-1])
    json.dump(d, open(f"profiles/{tag}_bench_{w}.json", "w"), indent=1)
    algo[d["config"]["workload"].split(" ")[0]] = d["roofline"]["algorithmic_bytes_per_launch"]
    print(f"{w:20s} {d['value']:.3e} nnz/s  {d['ms_per_step']:.3f} ms/step  frac {d['roofline']['frac']:.3f}  "
          f"gap {d['time_to_gap'] and d['time_to_gap'].get('seconds')}")
for rep in sorted(glob.glob(f"{src}/{tag}m_ncu_*.ncu-rep")):
    w = rep.split(f"{tag}m_ncu_")[1][:-8]
    subprocess.run([sys.executable, "scripts/ncu_summary.py", rep, f"profiles/{tag}_ncu_{w}.txt", "--json",
                    "profiles/ncu_traffic.json", "--workload", w] +
                   (["--algo-bytes", str(algo[w])] if w in algo else []), check=False,
                   stdout=subprocess.DEVNULL)
    print("summary", w)
lf = f"{src}/{tag}m_launches.csv"
if os.path.exists(lf):
    rows = [r for r in csv.reader(l for l in open(lf) if not l.startswith("=="))]
    h = rows[0]
    iK, iV = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        k = r[iK][:60]
        agg.setdefault(k, []).append(float(r[iV].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    out = ["# ncu --metrics gpu__time_duration.sum --clock-control none, nvtx range timed_steps of",
           "# python bench.py --no-gap --no-cpu --steps 3 --warmup 1 (default workload; cold-cache, serialised)",
           "launches  mean_us  share  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{len(v):8d} {sum(v) / len(v):9.1f} {100 * sum(v) / tot:5.1f}%  {k}")
    open(f"profiles/{tag}_launches.txt", "w").write("\n".join(out) + "\n")
    print("\n".join(out))
