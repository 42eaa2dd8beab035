#!/usr/bin/env python
"""Attribute an ncu source-page SASS export to CUDA source lines.

usage: ncu -i prof.ncu-rep --page source --csv --print-source sass > sass.csv
       nvdisasm -g -c <kernel cubin> > all.dis
       python tools/ncu_lines.py sass.csv all.dis <mangled kernel name> [file-substring]
Prints instructions executed and stall samples per source line (top lines) and per region."""
import csv
import re
import sys
from collections import defaultdict


def line_map(dis_path, fn, fsub):
    lines = open(dis_path).read().split("\n")
    start = None
    for i, l in enumerate(lines):
        if l.startswith(".text." + fn + ":"):
            start = i
            break
    if start is None:
        raise SystemExit("kernel not found in disassembly")
    cur = None
    m = {}
    for l in lines[start + 1:]:
        if l.startswith("//--------------------- .text.") or l.startswith(".section"):
            break
        g = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
        if g:
            cur = (g.group(1), int(g.group(2)))
            continue
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if a:
            off = int(a.group(1), 16)
            op = a.group(2).split()
            op = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "")
            m[off] = (cur, op)
    return m


def main():
    sass_csv, dis, fn = sys.argv[1:4]
    fsub = sys.argv[4] if len(sys.argv) > 4 else ".cu"
    m = line_map(dis, fn, fsub)
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    ia, ii, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    base = None
    per_line = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
    tot_i = tot_s = 0.0
    for r in rows[2:]:
        if len(r) <= max(ia, ii, iss):
            continue
        try:
            addr = int(r[ia], 16)
        except ValueError:
            continue
        if base is None:
            base = addr
        off = addr - base
        src, op = m.get(off, (None, "?"))
        key = f"{src[0].split('/')[-1]}:{src[1]}" if src else "?"
        ni = float(r[ii] or 0)
        ns = float(r[iss] or 0)
        per_line[key][0] += ni
        per_line[key][1] += ns
        per_line[key][2][op.split(".")[0]] += ni
        tot_i += ni
        tot_s += ns
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
    top = sorted(per_line.items(), key=lambda kv: -kv[1][1])[:45]
    print(f"{'line':28s} {'instr%':>7s} {'stall%':>7s}  top ops")
    for k, (ni, ns, ops) in top:
        o = sorted(ops.items(), key=lambda kv: -kv[1])[:4]
        print(f"{k:28s} {100*ni/tot_i:7.2f} {100*ns/tot_s:7.2f}  " +
              " ".join(f"{a}:{100*b/max(ni,1):.0f}%" for a, b in o))


if __name__ == "__main__":
    main()


def regions(sass_csv, dis, fn, spans):
    """spans: {name: [(file_substring, lo, hi), ...]} -> printed instruction / stall shares."""
    m = line_map(dis, fn, "")
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    ia, ii, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    base = None
    acc = defaultdict(lambda: [0.0, 0.0])
    ti = ts = 0.0
    for r in rows[2:]:
        try:
            addr = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        base = addr if base is None else base
        src, _ = m.get(addr - base, (None, "?"))
        ni, ns = float(r[ii] or 0), float(r[iss] or 0)
        ti += ni
        ts += ns
        name = "other"
        if src:
            for nm, sp in spans.items():
                if any(f in src[0] and lo <= src[1] <= hi for f, lo, hi in sp):
                    name = nm
                    break
        acc[name][0] += ni
        acc[name][1] += ns
    for k, (a, b) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:20s} instr {100*a/ti:6.2f}%  stall-samples {100*b/ts:6.2f}%")


def stall_regions(sass_csv, dis, fn, spans, kinds=("stall_wait", "stall_long_sb", "stall_barrier",
                                                    "stall_selected", "stall_not_selected",
                                                    "stall_math", "stall_short_sb")):
    """Per region: samples of each stall reason (share of all samples)."""
    m = line_map(dis, fn, "")
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    ia = hdr.index("Address")
    ik = [hdr.index(k) for k in kinds]
    base = None
    acc = defaultdict(lambda: [0.0] * len(kinds))
    tot = 0.0
    for r in rows[2:]:
        try:
            addr = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        base = addr if base is None else base
        src, _ = m.get(addr - base, (None, "?"))
        name = "other"
        if src:
            for nm, sp in spans.items():
                if any(f in src[0] and lo <= src[1] <= hi for f, lo, hi in sp):
                    name = nm
                    break
        for j, i in enumerate(ik):
            v = float(r[i] or 0)
            acc[name][j] += v
            tot += v
    print(f"{'region':16s} " + " ".join(f"{k.replace('stall_',''):>9s}" for k in kinds))
    for k, vals in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:16s} " + " ".join(f"{100*v/tot:9.2f}" for v in vals))
