#!/usr/bin/env python
"""Summarise an `ncu --page source --csv --print-source sass` export by opcode:
executed instructions, shared wavefronts vs ideal, stall samples (first kernel only)."""
import collections
import csv
import sys


def main(path, kernel_idx=0):
    rows = list(csv.reader(open(path)))
    sections, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            sections.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur and len(r) >= len(cur["hdr"]):
            cur["rows"].append(r)
    s = sections[kernel_idx]
    hdr = s["hdr"]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0, 0, 0])
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    stalls = collections.Counter()

    def num(x):
        try:
            return int(float(x))
        except ValueError:
            return 0

    for r in s["rows"]:
        src = r[ix["Source"]].strip().split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        op = op.split(".")[0]
        a = agg[op]
        a[0] += num(r[ix["Instructions Executed"]])
        a[1] += num(r[ix["L1 Wavefronts Shared"]])
        a[2] += num(r[ix["L1 Wavefronts Shared Ideal"]])
        a[3] += num(r[ix["Warp Stall Sampling (All Samples)"]])
        for c in stall_cols:
            stalls[c] += num(r[ix[c]])
    tot = sum(a[0] for a in agg.values()) or 1
    ts = sum(a[3] for a in agg.values()) or 1
    print(s["name"])
    for op, a in sorted(agg.items(), key=lambda x: -x[1][0])[:28]:
        print(f"  {op:10s} inst {a[0]:11d} ({100 * a[0] / tot:5.1f}%)  shared wf {a[1]:10d} ideal {a[2]:10d}"
              f"  stall samples {a[3]:7d} ({100 * a[3] / ts:5.1f}%)")
    print("  stall reasons:", ", ".join(f"{k[6:]}={100 * v / ts:.1f}%" for k, v in stalls.most_common(10)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
