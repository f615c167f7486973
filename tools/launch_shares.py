#!/usr/bin/env python
"""Per-segment share of a bench step: the ncu launch list (`ncu --metrics gpu__time_duration.sum
--clock-control none --csv --log-file L python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu`) against
the CUDA-event segments of a bench line from the same box.

  python tools/launch_shares.py --launches L.csv --bench bench.json --tag r02_final --out profiles/x.md

ncu times are cold-cache and serialised, so the SHARE of the step is what must agree, not the absolute.
The BCA backward segments include their dw finalize launch (rdfft2_kernel<float, p>)."""
import argparse
import csv
import io
import json
import statistics

SEGMENTS = {
    "bca_fwd_roberta_base": ["bca_fwd2_kernel"],
    "bca_fwd_llama2_7b": ["bca_fwd5_kernel"],
    "rdfft_fwd": ["rdfft2fo_kernel"],
    "packed_mul": ["packed_mul2_kernel"],
    "rdfft_inv": ["rdfft2o_inv_kernel"],
    "bca_bwd_roberta_base": ["bca_bwd3_kernel", "rdfft2_kernel<rdfft::Plan2<float, 256"],
    "bca_bwd_llama2_7b": ["bca_bwd5_kernel", "rdfft2_kernel<rdfft::Plan2<float, 1024"],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", required=True)
    ap.add_argument("--bench", required=True)
    ap.add_argument("--tag", default="")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    txt = open(a.launches).read().splitlines()
    start = [k for k, line in enumerate(txt) if line.startswith('"ID"')][0]
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(txt[start:])))
            if r.get("Metric Name") == "gpu__time_duration.sum"]

    def med(pat):
        v = [float(r["Metric Value"]) / 1e6 for r in rows if pat in r["Kernel Name"]]
        return statistics.median(v) if v else 0.0

    ev = json.load(open(a.bench))["segments_ms"]
    ncu = {k: sum(med(p) for p in pats) for k, pats in SEGMENTS.items()}
    tn, te = sum(ncu.values()), sum(ev[k] for k in SEGMENTS)
    out = [f"# ncu launch list of one bench step vs the CUDA-event segments ({a.tag})", "",
           "Median ncu time per launch of the step's kernels (cold-cache, serialised) and its share of the step, "
           "next to the bench line's CUDA-event segments and their share (`tools/launch_shares.py`).", "",
           "| segment | kernel(s) | ncu ms per launch | ncu share of step | CUDA-event ms | CUDA-event share |",
           "|---|---|---|---|---|---|"]
    for k, pats in SEGMENTS.items():
        names = " + ".join("`" + p.split("<")[0] + "`" for p in pats)
        out.append(f"| {k} | {names} | {ncu[k]:.4f} | {100 * ncu[k] / tn:.1f} % | {ev[k]:.4f} | {100 * ev[k] / te:.1f} % |")
    open(a.out, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
