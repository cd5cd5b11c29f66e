#!/usr/bin/env python
"""Per-kernel stall-reason totals and the top SASS lines of an `ncu --page source --csv` dump
(gzip ok).  Tool.   python tools/ncu_stalls.py gpurun_out/dev/full_source.csv.gz [ntop]"""
import csv
import gzip
import sys


def main():
    path = sys.argv[1]
    ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    kern, data, hdr = None, {}, None
    for r in rows:
        if len(r) >= 2 and r[0] == "Kernel Name":
            kern = r[1]
            data.setdefault(kern, [])
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if len(r) > 5 and r[0].startswith("0x"):
            data[kern].append(r)
    st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    for k, v in data.items():
        tot = sum(int(r[2]) for r in v) or 1
        print("==", k, len(v), "SASS lines,", tot, "samples")
        sums = {hdr[i]: sum(int(r[i] or 0) for r in v) for i in st}
        print("   ", ", ".join(f"{a[6:]} {b / tot * 100:.1f}%" for a, b in sorted(sums.items(), key=lambda x: -x[1]) if b / tot > 0.01))
        for idx, r in sorted(enumerate(v), key=lambda x: -int(x[1][2]))[:ntop]:
            why = max(st, key=lambda i: int(r[i] or 0))
            print(f"   {int(r[2]) / tot * 100:5.1f}%  [{idx:5d}] {r[1].strip()[:60]:60s} {hdr[why][6:]}")


if __name__ == "__main__":
    main()
