#!/usr/bin/env python
"""Map ncu per-SASS-instruction stall samples (--page source --csv) to CUDA source lines using
the line table of a local `nvdisasm -g -c` listing of the same build.  Tool.

  python tools/ncu_lines.py listing.sass full_source.csv.gz kernel_substring [ntop]
"""
import collections
import csv
import gzip
import re
import sys


def line_table(sass, kern):
    cur_fn, cur_line, table = None, None, {}
    for ln in open(sass):
        m = re.match(r"^\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = (m.group(1).rsplit("/", 1)[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m and cur_fn and kern in cur_fn:
            table[int(m.group(1), 16) // 16] = (cur_line, m.group(2).strip())
    return table


def main():
    sass, src, kern = sys.argv[1:4]
    ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    table = line_table(sass, kern)
    f = gzip.open(src, "rt") if src.endswith(".gz") else open(src)
    rows = list(csv.reader(f))
    cur, hdr, data, k = None, None, [], 0
    for r in rows:
        if len(r) >= 2 and r[0] == "Kernel Name":
            cur = r[1]
            k = 0
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if cur and kern in cur and len(r) > 5 and r[0].startswith("0x"):
            data.append((k, r))
            k += 1
    st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.defaultdict(lambda: [0, collections.Counter(), 0])
    tot = 0
    for idx, r in data:
        n = int(r[2] or 0)
        tot += n
        key = table.get(idx, (("?", 0), ""))[0]
        a = agg[key]
        a[0] += n
        a[2] += int(r[5] or 0)
        for i in st:
            a[1][hdr[i][6:]] += int(r[i] or 0)
    print(f"{kern}: {len(data)} SASS lines (listing {len(table)}), {tot} samples")
    for key, (n, why, ex) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:ntop]:
        top = ", ".join(f"{k} {v * 100 // max(n, 1)}%" for k, v in why.most_common(2))
        print(f"{n / max(tot, 1) * 100:5.1f}%  {key[0]}:{key[1]:<5d} inst {ex:>11d}  {top}")


if __name__ == "__main__":
    main()
