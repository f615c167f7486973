#!/usr/bin/env python
"""Build check: compile every translation unit of librdfft.so with `ptxas -v` and
fail if any kernel spills registers to local memory (every instantiated kernel is on a dispatched
path: the dispatch instantiates nothing it cannot launch).

  python tools/check_spills.py            # exit 1 and list the kernels if any spill
"""
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01385_b200 import build as B  # noqa: E402


def ptxas_report(src):
    cmd = [B.NVCC, *B.FLAGS, "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-c", "-o", os.devnull, src]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode:
        raise RuntimeError(out.stderr[-2000:])
    rows, cur = [], None
    for line in out.stderr.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            rows.append((cur, int(m.group(1)), int(m.group(2)), int(m.group(3))))
        m = re.search(r"Used (\d+) registers", line)
        if m and rows and rows[-1][0] == cur and len(rows[-1]) == 4:
            rows[-1] = rows[-1] + (int(m.group(1)),)
    return rows


def main():
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        reports = list(ex.map(ptxas_report, B.sources()))
    bad = []
    n = 0
    for rows in reports:
        for r in rows:
            n += 1
            if r[2] or r[3]:
                bad.append(r)
    for r in bad:
        print(f"SPILL {r[2]} B st / {r[3]} B ld, stack {r[1]} B, regs {r[4] if len(r) > 4 else '?'}: {r[0]}")
    print(f"{n} kernels, {len(bad)} with spills")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
