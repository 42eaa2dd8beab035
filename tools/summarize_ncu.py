#!/usr/bin/env python
"""Summarise an ncu capture of k_tile and a launch list into profiles/ (tracked).

usage: python tools/summarize_ncu.py <tag> <prof.ncu-rep> <launches.csv> [bench.json]
writes profiles/<tag>_k_tile.md, profiles/<tag>_launches.csv, profiles/traffic_<config>.json
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = [
    "gpu__time_duration.sum", "gpc__cycles_elapsed.max", "sm__cycles_active.avg",
    "sm__cycles_active.min", "sm__cycles_active.max", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
]


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    tot = collections.Counter()
    mix = collections.Counter()
    texec = 0.0
    for r in rows[2:]:
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    tot[h] += float(r[ix[h]].replace(",", "") or 0)
                except ValueError:
                    pass
        try:
            e = float(r[ix["Instructions Executed"]].replace(",", "") or 0)
        except ValueError:
            e = 0.0
        texec += e
        op = r[ix["Source"]].split()
        if op:
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            mix[o.split(".")[0]] += e
    s = sum(tot.values()) or 1.0
    return ({k: round(100 * v / s, 1) for k, v in tot.most_common(8)},
            {k: round(100 * v / texec, 1) for k, v in mix.most_common(12)}, texec)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg, cnt = collections.OrderedDict(), collections.Counter()
    for r in data:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0][:80]
        v = float(r[vi].replace(",", ""))
        v *= {"msecond": 1e6, "usecond": 1e3}.get(r[ui], 1.0)
        agg[k] = agg.get(k, 0.0) + v
        cnt[k] += 1
    return agg, cnt


def main():
    tag, rep, lcsv = sys.argv[1], sys.argv[2], sys.argv[3]
    bench = json.load(open(sys.argv[4])) if len(sys.argv) > 4 else None
    raw = ncu_raw(rep)
    st, mix, texec = stalls(rep)
    agg, cnt = launches(lcsv)
    tot = sum(agg.values())
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary `{tag}` — k_tile (full set, --clock-control none)", ""]
    if bench:
        lines += [f"bench: `{bench['config']['workload']}` value {bench['value']:.4g} px/s, "
                  f"{bench['ms_per_step']:.2f} ms/step, k_tile {bench['roofline']['tile_kernel_ms_per_step']:.2f} ms "
                  f"(live CUDA events), frac {bench['roofline']['frac']:.3f} of {bench['roofline']['peak']:.1f} "
                  f"{bench['roofline']['unit']}", ""]
    lines += ["| metric | value | unit |", "|---|---|---|"]
    for k in WANT:
        if k in raw:
            lines.append(f"| {k} | {raw[k][0]} | {raw[k][1]} |")
    lines += ["", "warp-stall mix (% of samples): " + ", ".join(f"{k[6:]} {v}" for k, v in st.items()),
              "", "instruction mix (% of executed): " + ", ".join(f"{k} {v}" for k, v in mix.items()),
              "", f"executed warp instructions: {texec:.4g}", "",
              "## launch list share (ncu, serialised, cold-cache; compare shares)", "",
              "| kernel | total ms | share | launches |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:15]:
        lines.append(f"| `{k}` | {v / 1e6:.3f} | {100 * v / tot:.1f}% | {cnt[k]} |")
    with open(os.path.join(ROOT, "profiles", f"{tag}_k_tile.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    # per-launch DRAM traffic of the captured k_tile launch
    def num(k):
        v, u = raw[k]
        return float(v.replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
    traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    cfg = bench["config"]["workload"].split(":")[0] if bench else tag.split("_")[-1]
    with open(os.path.join(ROOT, "profiles", f"traffic_{cfg}.json"), "w") as f:
        json.dump({"k_tile_dram_bytes_per_launch": traffic, "source": f"profiles/{tag}_k_tile.md"}, f)
    subprocess.run(["cp", lcsv, os.path.join(ROOT, "profiles", f"{tag}_launches.csv")], check=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
