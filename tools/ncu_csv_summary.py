#!/usr/bin/env python
"""Summarise `ncu --page raw --csv` + `--page source --csv --print-source sass` exports (the .ncu-rep
files stay on the GPU box: gpurun copies back at most 64 MiB) into a markdown table for profiles/:

  python tools/ncu_csv_summary.py --raw A_raw.csv --sass A_sass.csv --units 16384 --unit-name token \
      [--raw B_raw.csv --sass B_sass.csv --units ...] --title "..." --out profiles/r02_x.md [--traffic-key k ...]

Per kernel: time, launch shape, registers, issue-active %, warps active %, FMA / ALU / LSU pipe %, shared
wavefronts (total, per unit, excess over ideal from the source page), bank conflicts, local loads/stores,
DRAM bytes, the top warp-stall reasons (per issue), and the SASS opcode mix with stall-sample shares.
"""
import argparse
import collections
import csv
import json
import re

RAW = {
    "gpu__time_duration.sum": "time",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wf",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed": "smem_wf_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "bank_ld",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "bank_st",
    "sass__inst_executed_local_loads": "local_ld",
    "sass__inst_executed_local_stores": "local_st",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "smsp__inst_executed.sum": "warp_inst",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "s": 1, "second": 1}


def read_raw(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units = rows[i], rows[i + 1]
    out = []
    for vals in rows[i + 2:]:
        d = dict(zip(hdr, vals))
        e = {"kernel": d["Kernel Name"], "stalls": {}}
        for h, u, v in zip(hdr, units, vals):
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            if h in RAW:
                e[RAW[h]] = x * SCALE.get(u, 1)
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
            if m:
                e["stalls"][m.group(1)] = x
        out.append(e)
    return out


def read_sass(path):
    kern, cur, hdr = {}, None, None
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "Kernel Name":
            cur, hdr = row[1], None
            kern[cur] = []
            continue
        if row[0] == "Address":
            hdr = row
            continue
        if hdr and cur:
            kern[cur].append(dict(zip(hdr, row)))
    res = {}
    for name, rows in kern.items():
        mix, stall = collections.Counter(), collections.Counter()
        wf = wf_ideal = 0
        for r in rows:
            ins = r.get("Source", "").strip()
            op = re.sub(r"^@!?U?P\w+\s+", "", ins).split(" ")[0].split(".")[0]
            n = int(float(r.get("Instructions Executed") or 0))
            mix[op] += n
            stall[op] += int(float(r.get("Warp Stall Sampling (All Samples)") or 0))
            wf += int(float(r.get("L1 Wavefronts Shared") or 0))
            wf_ideal += int(float(r.get("L1 Wavefronts Shared Ideal") or 0))
        res[name] = {"mix": mix, "stall": stall, "wf": wf, "wf_ideal": wf_ideal}
    return res


def short(name):
    name = name.replace("rdfft::", "").replace("void ", "").replace("(int)", "").replace("(bool)", "")
    depth, cut = 0, len(name)
    for i, ch in enumerate(name):  # drop the argument list: the first "(" outside the template brackets
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            cut = i
            break
    return name[:cut].strip()


def match(sass, kernel):
    for k, v in sass.items():
        if short(k) == short(kernel):
            return v
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--raw", action="append", required=True)
    ap.add_argument("--sass", action="append", default=[])
    ap.add_argument("--units", action="append", type=float, default=[])
    ap.add_argument("--unit-name", action="append", default=[])
    ap.add_argument("--title", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic", help="update this ncu_traffic.json with --traffic-key entries")
    ap.add_argument("--traffic-key", action="append", default=[], help="KEY=kernel-regex[@batch]")
    a = ap.parse_args()
    md = [f"# {a.title}\n"]
    table = ["| kernel | grid x block | regs | us | issue % | warps % | FMA % | ALU % | LSU % | shared wavefronts "
             "(per unit; excess) | bank conflicts ld/st | local ld/st | DRAM R+W MB |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    detail = []
    allk = []
    for i, rp in enumerate(a.raw):
        sass = read_sass(a.sass[i]) if i < len(a.sass) else {}
        units = a.units[i] if i < len(a.units) else 0
        uname = a.unit_name[i] if i < len(a.unit_name) else "unit"
        for e in read_raw(rp):
            s = match(sass, e["kernel"])
            allk.append(e)
            wf = e.get("smem_wf", 0)
            per = f"{wf / units:.0f}/{uname}" if units else "-"
            exc = f"{(s['wf'] - s['wf_ideal']) / max(s['wf'], 1) * 100:.0f}%" if s and s["wf"] else "-"
            table.append(
                f"| `{short(e['kernel'])}` | {int(e.get('grid', 0))} x {int(e.get('block', 0))} | {int(e.get('regs', 0))} | "
                f"{e.get('time', 0) * 1e6:.1f} | {e.get('issue_pct', 0):.1f} | {e.get('warps_pct', 0):.1f} | "
                f"{e.get('fma_pct', 0):.1f} | {e.get('alu_pct', 0):.1f} | {e.get('lsu_pct', 0):.1f} | "
                f"{wf / 1e6:.2f} M ({per}; {exc}) | {int(e.get('bank_ld', 0))}/{int(e.get('bank_st', 0))} | "
                f"{int(e.get('local_ld', 0))}/{int(e.get('local_st', 0))} | "
                f"{(e.get('dram_rd', 0) + e.get('dram_wr', 0)) / 1e6:.1f} |")
            st = sorted(e["stalls"].items(), key=lambda kv: -kv[1])[:8]
            detail.append(f"### `{short(e['kernel'])}`\n")
            wi = e.get("warp_inst", 0)
            detail.append(f"- warp instructions: {wi / 1e6:.2f} M" + (f" ({wi / units:.0f} per {uname})" if units else ""))
            detail.append("- top stalls (warps per issue): " + ", ".join(f"{k} {v:.2f}" for k, v in st))
            if s:
                tot = sum(s["mix"].values()) or 1
                ss = sum(s["stall"].values()) or 1
                detail.append("- SASS mix (share of executed warp instructions / of stall samples): " + ", ".join(
                    f"{op} {100 * n / tot:.1f}%/{100 * s['stall'][op] / ss:.1f}%" for op, n in s["mix"].most_common(14)))
                detail.append(f"- shared wavefronts from the source page: {s['wf'] / 1e6:.2f} M, ideal "
                              f"{s['wf_ideal'] / 1e6:.2f} M")
            detail.append("")
    md += table + [""] + detail
    open(a.out, "w").write("\n".join(md) + "\n")
    print("\n".join(md))
    if a.traffic:
        try:
            tr = json.load(open(a.traffic))
        except (OSError, ValueError):
            tr = {}
        for spec in a.traffic_key:
            key, rx = spec.split("=", 1)
            batch = None
            if "@" in rx:
                rx, batch = rx.split("@")
            for e in allk:
                if re.search(rx, e["kernel"]):
                    tr[key] = {"dram_bytes_per_launch": e.get("dram_rd", 0) + e.get("dram_wr", 0),
                               "kernel": short(e["kernel"]), "duration_s": e.get("time"), "source": a.out}
                    if batch:
                        tr[key]["batch"] = int(batch)
                    break
        json.dump(tr, open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
