#!/usr/bin/env python
"""Summarise an ncu report of the fused kernel into profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_fused_converged.txt \
        [--json profiles/ncu_traffic.json --workload 1M_x_10k --algo-bytes N]
"""
import argparse
import collections
import csv
import json
import re
import subprocess


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--json")
    ap.add_argument("--workload", default="1M_x_10k")
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rows = ncu_csv(a.rep, "--page", "details")
    h = rows[0]
    keep = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
            "Issue Slots Busy", "Executed Instructions", "Registers Per Thread", "Achieved Occupancy",
            "L1/TEX Hit Rate", "L2 Hit Rate", "Eligible Warps Per Scheduler", "No Eligible",
            "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
    lines = [f"# ncu --set full summary: {a.rep}", a.note, ""]
    kname = None
    for r in rows[1:]:
        d = dict(zip(h, r))
        kname = d.get("Kernel Name", kname)
        if d.get("Metric Name") in keep:
            lines.append(f"{d['Metric Name']:34s} {d['Metric Value']} {d['Metric Unit']}")
    raw = ncu_csv(a.rep, "--page", "raw")
    rd = dict(zip(raw[0], raw[2])) if len(raw) > 2 else {}
    def num(k):
        try:
            return float(rd[k].replace(",", ""))
        except (KeyError, ValueError):
            return None
    unit = raw[1][raw[0].index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in raw[0] else ""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    rb, wb = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    wunit = raw[1][raw[0].index("dram__bytes_write.sum")] if "dram__bytes_write.sum" in raw[0] else ""
    wscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(wunit, 1)
    traffic = (rb or 0) * scale + (wb or 0) * wscale
    lines += ["", f"kernel: {kname}", f"dram__bytes_read.sum + dram__bytes_write.sum = {traffic:.6g} bytes per launch"]
    if a.algo_bytes:
        lines.append(f"algorithmic bytes per launch = {a.algo_bytes:.6g}  (traffic / algorithmic = {traffic / a.algo_bytes:.3f})")
    # stall reasons and hottest source lines
    src = ncu_csv(a.rep, "--page", "source", "--print-source", "cuda,sass")
    if len(src) > 3:
        hdr = src[2]
        iIE = hdr.index("Instructions Executed")
        stall_cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
        agg, st = collections.Counter(), collections.Counter()
        text = {}
        cur = None
        for r in src[3:]:
            if len(r) < len(hdr):
                continue
            if r[0] != "":
                cur = r[0]
                text[cur] = r[1].strip()[:100]
            try:
                agg[cur] += int(r[iIE])
                for i in stall_cols:
                    st[hdr[i]] += int(r[i] or 0)
            except ValueError:
                pass
        tot, tst = sum(agg.values()) or 1, sum(st.values()) or 1
        lines += ["", "stall reasons: " + ", ".join(f"{k[6:]} {v / tst * 100:.1f}%" for k, v in st.most_common(8)),
                  "", "hottest source lines (share of executed instructions):"]
        for k, v in agg.most_common(25):
            lines.append(f"  {v / tot * 100:5.1f}%  L{k}: {text.get(k, '')}")
    open(a.out, "w").write("\n".join(lines) + "\n")
    if a.json:  # per-workload map read by bench.py (roofline.traffic)
        try:
            table = json.load(open(a.json))
        except (OSError, ValueError):
            table = {}
        table[a.workload] = {"kernel": kname, "dram_bytes_per_launch": traffic, "report": a.rep,
                             "summary": a.out, "algorithmic_bytes_per_launch": a.algo_bytes}
        json.dump(table, open(a.json, "w"), indent=1, sort_keys=True)
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    main()
