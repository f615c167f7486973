#!/usr/bin/env python
"""Summarise ncu captures for profiles/:

  python tools/ncu_summary.py --reps gpurun_out/TAG/prof_*.ncu-rep --launches gpurun_out/TAG/launches.csv \
      --bench gpurun_out/TAG/bench.json --out profiles/TAG

writes <out>.md (human summary) and <out>_traffic.json (dram bytes per launch per kernel, consumed by
bench.py's roofline.traffic via profiles/ncu_traffic.json).
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "bank_conf_ld",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "bank_conf_st",
    "sass__inst_executed_local_loads": "local_ld",
    "sass__inst_executed_local_stores": "local_st",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_inst",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                d[KEYS[h]] = x * SCALE.get(u, 1)
        res.append(d)
    return res


def short(name):
    m = re.search(r"(rdfft\w*kernel|bca_\w+kernel|packed_mul_kernel|\w+_kernel)", name)
    base = m.group(1) if m else name[:40]
    t = re.search(r"<(.*)>", name)
    return base + ("<" + t.group(1)[:60] + ">" if t else "")


def family(name):
    if "rdfft2o_inv_kernel" in name:
        return "rdfft_inv"
    if "rdfft2_kernel" in name:
        if re.search(r"<float,", name) and re.search(r",\s*(?:true|\(bool\)1|1)>\s*(?:\(|$)", name):
            return "bca_bwd"  # the bench's only fp32 transform: bca_bwd's in-place dw finalize
        return "rdfft_inv" if re.search(r",\s*(?:true|\(bool\)1|1)>\s*(?:\(|$)", name) else "rdfft_fwd"
    for k, f in [("bca_fwd", "bca_fwd"), ("bca_bwd", "bca_bwd"), ("packed_mul", "packed_mul"),
                 ("rdfft2_kernel", "rdfft"), ("rdfft_v1", "rdfft_v1")]:
        if k in name:
            return f
    return "other"


def launches(path):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1)
        k = short(r["Kernel Name"])
        tot[k] += v
        cnt[k] += 1
    return tot, cnt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", nargs="*", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--bench")
    ap.add_argument("--out", required=True)
    ap.add_argument("--batch", type=int, default=1 << 18, help="vectors per transform launch in the captures")
    a = ap.parse_args()
    md = [f"# ncu summary: {os.path.basename(a.out)}\n"]
    traffic = {}
    if a.bench and os.path.exists(a.bench):
        b = json.loads(open(a.bench).read().strip().splitlines()[-1])
        md.append("## bench line (CUDA events, not under ncu)\n")
        md.append(f"- value: {b['value']:.1f} {b['unit']} ({100 * b.get('frac_of_hbm_peak', 0):.1f}% of the bench peak)")
        md.append(f"- segments (ms per step): " + ", ".join(f"{k} {v:.3f}" for k, v in b["segments_ms"].items()))
        md.append(f"- clocks: {b.get('clocks')}\n")
    if a.launches and os.path.exists(a.launches):
        tot, cnt = launches(a.launches)
        s = sum(tot.values())
        # the bench's own kernels (input generation by torch runs before the timed region)
        ours = sum(v for k, v in tot.items() if family(k) != "other")
        md.append("## launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)\n")
        md.append("Shares: of every launch in the process, and of the step (this library's kernels only; the "
                  "torch kernels generate the inputs before the timed region).\n")
        md.append("| kernel | launches | total us | share (all) | share of step |\n|---|---|---|---|---|")
        fam_ncu = collections.defaultdict(float)
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            fam = family(k)
            step_share = f"{100 * v / ours:.1f}%" if fam != "other" and ours > 0 else "-"
            if fam != "other":
                fam_ncu[fam] += v
            md.append(f"| `{k}` | {cnt[k]} | {v * 1e6:.1f} | {100 * v / s:.1f}% | {step_share} |")
        md.append("")
        if a.bench and os.path.exists(a.bench) and ours > 0:
            seg = b["segments_ms"]
            tseg = sum(seg.values())
            md.append("Share of the step per kernel: ncu launch list (cold, serialised) vs the bench's CUDA events\n")
            md.append("| kernel | ncu share | CUDA-event share |\n|---|---|---|")
            for fam in seg:
                md.append(f"| {fam} | {100 * fam_ncu.get(fam, 0) / ours:.1f}% | {100 * seg[fam] / tseg:.1f}% |")
            md.append("")
    md.append("## full captures (`ncu --set full`, one launch each)\n")
    md.append("| kernel | grid x block | regs | us | DRAM R+W MB | DRAM % | issue % | occupancy % | "
              "smem bank conflicts ld/st | local ld/st |\n|---|---|---|---|---|---|---|---|---|---|")
    for rep in a.reps:
        for d in raw(rep):
            fam = family(d["kernel"])
            t = d.get("dram_read", 0) + d.get("dram_write", 0)
            traffic.setdefault(fam, {"dram_bytes_per_launch": t, "kernel": short(d["kernel"]),
                                     "duration_s": d.get("duration"), "source": os.path.basename(rep),
                                     "batch": a.batch})
            md.append(f"| `{short(d['kernel'])}` | {int(d.get('grid', 0))} x {int(d.get('block', 0))} | "
                      f"{int(d.get('regs', 0))} | {d.get('duration', 0) * 1e6:.1f} | {t / 1e6:.1f} | "
                      f"{d.get('dram_pct', 0):.1f} | {d.get('issue_pct', 0):.1f} | {d.get('occupancy_pct', 0):.1f} | "
                      f"{int(d.get('bank_conf_ld', 0))}/{int(d.get('bank_conf_st', 0))} | "
                      f"{int(d.get('local_ld', 0))}/{int(d.get('local_st', 0))} |")
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(md) + "\n")
    with open(a.out + "_traffic.json", "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
